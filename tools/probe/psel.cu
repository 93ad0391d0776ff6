// Probe: per-step timeline of the TSLU select (one CTA), using select.cuh's trace points.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRLHC_SEL_TRACE -o psel psel.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2412_06551_b200/csrc/select.cuh"
using namespace rlhc;
constexpr int W = 64, NW = 8, RS = 8, CW = W / NW;
__device__ long long* g_trace;

__global__ void __launch_bounds__(256, 1) k_sel(const double* vals, int* out) {
  extern __shared__ __align__(16) unsigned char raw[];
  SelSmem<W, NW, RS>& sm = *reinterpret_cast<SelSmem<W, NW, RS>*>(raw);
  sel_init(sm);
  const int lane = lane_id(), wp = warp_id();
  double a[RS][CW];
  int gid[RS];
  unsigned act = 0;
  for (int s = 0; s < RS; s++) {
    int r = s * 32 + lane;
    gid[s] = r;
    act |= 1u << s;
    for (int c = 0; c < CW; c++) a[s][c] = vals[r * W + wp + NW * c];
  }
  for (int i = threadIdx.x; i < 65 * 32; i += blockDim.x) sm.trace[i] = 0;
  __syncthreads();
  SEL_TRACE(0)
  int steps = gepp_select<W, NW, RS>(a, act, gid, W, sm);
  SEL_TRACE(64 * 32 + 1)
  __syncthreads();
  for (int i = threadIdx.x; i < 65 * 32; i += blockDim.x) g_trace[i] = sm.trace[i];
  if (threadIdx.x < W) out[threadIdx.x] = sm.out_id[threadIdx.x] + steps * 0;
}

int main() {
  const int R = 32 * RS;
  std::vector<double> h(R * W);
  srand(1);
  for (auto& v : h) v = (double)rand() / RAND_MAX - 0.5;
  double* d; int* o; long long* tr;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 256 * 4); cudaMalloc(&tr, 65 * 32 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr));
  int smem = sizeof(SelSmem<W, NW, RS>);
  cudaFuncSetAttribute(k_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int it = 0; it < 3; it++) {
    cudaMemset(tr, 0, 65 * 32 * 8);
    k_sel<<<1, 256, smem>>>(d, o);
    cudaDeviceSynchronize();
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> t(65 * 32);
  cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
  long long t0 = t[0];
  printf("total %lld cycles (%.0f per step)\n", t[64 * 32 + 1] - t0, (t[64 * 32 + 1] - t0) / 64.0);
  for (int s = 0; s < 64; s++) {
    int q = s % NW;
    long long* r = &t[s * 32];
    // owner: wake (2q), pivot start (16), keys+tree (->18), redux hi (->19), lo (->20),
    // ballots (->21), publish (->22), pivot end (17), done (2q+1)
    printf("t=%2d own=%d wake=%6lld piv0=%6lld tree=%4lld rhi=%4lld rlo=%4lld minidx=%4lld pub=%4lld end=%4lld done=%6lld | ",
           s, q, r[2 * q] ? r[2 * q] - t0 : -1, r[16] - t0, r[18] - r[16], r[19] - r[18], r[20] - r[19],
           r[21] - r[20], r[22] - r[21], r[17] - r[22], r[2 * q + 1] - t0);
    for (int w = 0; w < NW; w++) printf("%6lld ", r[2 * w + 1] ? r[2 * w + 1] - t0 : -1);
    printf("\n");
  }
}
