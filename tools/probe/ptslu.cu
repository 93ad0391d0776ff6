// Probe: phase timeline (globaltimer) of the TSLU leaf and node kernels at cfg2's shape
// (65536 x 64, 256-row leaves, arity 4): per block, load / select / output, and the gaps
// between back-to-back levels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRLHC_TSLU_TRACE -o ptslu ptslu.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include "../../paper_2412_06551_b200/csrc/tslu.cu"
namespace rlhc {
void note_launch() {}
}
using namespace rlhc;

int main() {
  const int m = 65536, n = 64, W = 64, leaf = 256, arity = 4;
  std::vector<double> h((size_t)m * n);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = nd(g);
  double* X; cudaMalloc(&X, h.size() * 8);
  cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  int nleaves = m / leaf;
  int *ids[2], *cnt[2]; double* vals[2];
  for (int k = 0; k < 2; k++) {
    cudaMalloc(&ids[k], nleaves * W * 4); cudaMalloc(&cnt[k], nleaves * 4); cudaMalloc(&vals[k], (size_t)nleaves * W * W * 8);
  }
  cudaStream_t st; cudaStreamCreate(&st);
  const int base[5] = {0, 256, 320, 336, 340}, nb[5] = {256, 64, 16, 4, 1};
  for (int rep = 0; rep < 4; rep++) {
    // the library's single-process mode: ids-only slots, nodes read rows of X by id
    const RowSrc rsrc{X, n, 0, 0};
    launch_tslu_leaf(W, X, n, m, 0, 0, n, nullptr, ids[0], cnt[0], nullptr, st, nullptr, nullptr);
    int cur = 0, ns = nleaves;
    while (ns > 1) {
      int nout = (ns + arity - 1) / arity;
      launch_tslu_node(W, ids[cur], cnt[cur], nullptr, ns, arity, n, ids[cur ^ 1], cnt[cur ^ 1], nullptr, st, nullptr,
                       &rsrc);
      ns = nout; cur ^= 1;
    }
    cudaStreamSynchronize(st);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  std::vector<unsigned long long> t(4096 * 8);
  cudaMemcpyFromSymbol(t.data(), g_tslu_trace, t.size() * 8);
  unsigned long long T0 = ~0ull;
  for (int b = 0; b < 341; b++) T0 = std::min(T0, t[b * 8]);
  unsigned long long prev_end = 0;
  for (int l = 0; l < 5; l++) {
    unsigned long long s0 = ~0ull, s1 = 0, e1 = 0;
    double ld = 0, so = 0, sel = 0, out = 0;
    for (int b = base[l]; b < base[l] + nb[l]; b++) {
      auto* r = &t[b * 8];
      s0 = std::min(s0, r[0]); s1 = std::max(s1, r[0]); e1 = std::max(e1, r[4]);
      if (l > 0) so += r[1] - r[0];
      ld += r[2] - (l > 0 ? r[1] : r[0]); sel += r[3] - r[2]; out += r[4] - r[3];
    }
    printf("level %d blocks %3d: start %7.1f (last start %7.1f) end %7.1f us | gap %5.1f us | per block: sort %.1f load %.1f select %.1f output %.1f us\n",
           l, nb[l], (s0 - T0) * 1e-3, (s1 - T0) * 1e-3, (e1 - T0) * 1e-3, l ? (double)(s0 - prev_end) * 1e-3 : 0.0,
           so / nb[l] * 1e-3, ld / nb[l] * 1e-3, sel / nb[l] * 1e-3, out / nb[l] * 1e-3);
    prev_end = e1;
  }
}
