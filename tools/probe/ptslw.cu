// Probe: per-warp phase timeline of the warp tournament (tslw.cu) at a given shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRLHC_TSLW_TRACE -o ptslw ptslw.cu
//   ./ptslw [m] [n]
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <tuple>
#include <vector>
#include "../../paper_2412_06551_b200/csrc/tslw.cu"
namespace rlhc {
void note_launch() {}
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return nullptr; }
cudaError_t launch_ts_gemm_checked(const double*, int64_t, double*, int64_t, const double*, int64_t, const double*,
                                   int64_t, int64_t, int, int, double*, unsigned long long*, int, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}
using namespace rlhc;

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 65536;
  const int n = argc > 2 ? atoi(argv[2]) : 64;
  std::vector<double> h((size_t)m * n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = nd(g);
  double *X, *Lb, *U, *L11, *rd, *lw;
  cudaMalloc(&X, h.size() * 8);
  cudaMalloc(&Lb, h.size() * 8);
  cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&U, (size_t)n * n * 8); cudaMalloc(&L11, (size_t)n * n * 8); cudaMalloc(&rd, n * 8); cudaMalloc(&lw, 256 * 8);
  int64_t* piv; cudaMalloc(&piv, n * 8);
  uint8_t* chosen; cudaMalloc(&chosen, m);
  unsigned long long* status; cudaMalloc(&status, 8); cudaMemset(status, 0xff, 8);
  int *ids[2], *cnt[2];
  double* vals[2];
  size_t ns = tslw_slots(m);
  for (int k = 0; k < 2; k++) {
    cudaMalloc(&ids[k], ns * 16 * 4); cudaMalloc(&cnt[k], (2 * ns + 64) * 4); cudaMalloc(&vals[k], ns * 256 * 8);
  }
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; rep++) {
    unsigned z = 0;
    cudaMemcpyToSymbol(g_twn, &z, 4);
    cudaMemcpyToSymbol(g_lvn, &z, 4);
    cudaEventRecord(e0, st);
    run_tslw(X, n, m, 0, n, 8, Lb, n, piv, U, L11, rd, lw, chosen, ids, cnt, vals, status, true, st);
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %.1f us\n", rep, ms * 1e3);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  {
    long long stp[64];
    cudaMemcpyFromSymbol(stp, g_stp, sizeof(stp));
    printf("per-step cycles (block 0 warp 0, last select):");
    for (int i = 1; i <= 16; i++) printf(" %lld", stp[i] - stp[i - 1]);
    printf("\n");
  }
  unsigned nrec; cudaMemcpyFromSymbol(&nrec, g_twn, 4);
  std::vector<unsigned long long> t((size_t)nrec * 8);
  cudaMemcpyFromSymbol(t.data(), g_tw, t.size() * 8);
  // per panel: phase-1 cycles (mean, max), select+climb cycles (mean, max), timeline
  std::map<unsigned long long, std::vector<unsigned long long*>> gr;
  unsigned long long T0 = ~0ull;
  for (unsigned i = 0; i < nrec && i < (1u << 16); i++) { gr[t[i * 8 + 1]].push_back(&t[i * 8]); T0 = std::min(T0, t[i * 8 + 3]); }
  for (auto& [k, v] : gr) {
    unsigned long long s0 = ~0ull, e = 0; double a = 0, b = 0, am = 0, bm = 0;
    for (auto* r : v) { s0 = std::min(s0, r[3]); e = std::max(e, r[7]); a += r[4]; b += r[5]; am = std::max(am, (double)r[4]); bm = std::max(bm, (double)r[5]); }
    printf("p0 %3llu warps %5zu: start %8.2f end %8.2f us | phase1 cycles mean %7.0f max %7.0f | select+climb mean %7.0f max %7.0f\n",
           k, v.size(), (s0 - T0) * 1e-3, (e - T0) * 1e-3, a / v.size(), am, b / v.size(), bm);
  }
  unsigned nl; cudaMemcpyFromSymbol(&nl, g_lvn, 4);
  std::vector<unsigned long long> lv((size_t)std::min(nl, 1u << 14) * 6);
  cudaMemcpyFromSymbol(lv.data(), g_lv, lv.size() * 8);
  std::map<std::pair<unsigned long long, unsigned long long>, std::vector<unsigned long long*>> lg;
  for (size_t i = 0; i < lv.size() / 6; i++) lg[{lv[i * 6], lv[i * 6 + 1]}].push_back(&lv[i * 6]);
  for (auto& [k, v] : lg) {
    double sel = 0, arr = 0, stg = 0, sm = 0, am = 0, gm = 0;
    for (auto* r : v) {
      sel += r[3] - r[2]; arr += r[4] - r[3]; stg += r[5] - r[4];
      sm = std::max(sm, (double)(r[3] - r[2])); am = std::max(am, (double)(r[4] - r[3])); gm = std::max(gm, (double)(r[5] - r[4]));
    }
    printf("p0 %3llu level %3llu warps %5zu: select %.2f (max %.2f) us, emit+arrive %.2f (max %.2f), node load %.2f (max %.2f)\n",
           k.first, k.second, v.size(), sel / v.size() * 1e-3, sm * 1e-3, arr / v.size() * 1e-3, am * 1e-3,
           stg / v.size() * 1e-3, gm * 1e-3);
  }
  return 0;
}
