// Latency of one leaf select (tslw.cu select_and_emit: 128 x 16 GEPP winners) with W select
// warps per SM and nothing else running: cycles per select.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o psel_lat psel_lat.cu
#include <cstdio>
#include <vector>
#include "../../paper_2412_06551_b200/csrc/tslw.cu"
namespace rlhc {
void note_launch() {}
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return nullptr; }
cudaError_t launch_ts_gemm_checked(const double*, int64_t, double*, int64_t, const double*, int64_t, const double*,
                                   int64_t, int64_t, int, int, double*, unsigned long long*, int, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
__global__ void sel_lat(int reps, int* ids, int* cnt, double* vals, long long* cyc, unsigned seed) {
  extern __shared__ __align__(16) unsigned char raw3[];
  WSel& sm = reinterpret_cast<WSel*>(raw3)[warp_id()];
  const int lane = lane_id();
  unsigned x = seed ^ (blockIdx.x * 977 + threadIdx.x * 131);
  for (int i = lane; i < WR * TS; i += 32) {
    x = x * 1664525u + 1013904223u;
    sm.tile[i] = (double)(int)(x >> 8) * 1e-6;
  }
  for (int s = 0; s < RS; s++) { sm.sid[s * 32 + lane] = s * 32 + lane; sm.rank[s * 32 + lane] = s * 32 + lane; }
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    const int slot = (blockIdx.x * blockDim.x / 32 + warp_id()) * reps + r;
    select_and_emit(sm, 0xfu, WW, slot, ids, cnt, vals, TslwRoot{}, 0);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + warp_id()] = (t1 - t0) / reps;
}
}
int main() {
  using namespace rlhc;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 64;
  for (int w : {1, 2, 4, 8}) {
    int *ids, *cnt; double* vals; long long* cyc;
    const int nw = sms * w;
    cudaMalloc(&ids, (size_t)nw * reps * WW * 4); cudaMalloc(&cnt, (size_t)nw * reps * 4);
    cudaMalloc(&vals, (size_t)nw * reps * WW * WW * 8); cudaMalloc(&cyc, nw * 8);
    cudaFuncSetAttribute(sel_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(w * sizeof(WSel)));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    sel_lat<<<sms, 32 * w, w * sizeof(WSel)>>>(2, ids, cnt, vals, cyc, 1);
    cudaEventRecord(a);
    sel_lat<<<sms, 32 * w, w * sizeof(WSel)>>>(reps, ids, cnt, vals, cyc, 7);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(nw); cudaMemcpy(h.data(), cyc, nw * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto v : h) avg += v; avg /= nw;
    printf("{\"select_warps_per_sm\":%d,\"cycles_per_select\":%.0f,\"us_per_select\":%.2f,\"selects_per_us_per_sm\":%.3f,\"err\":\"%s\"}\n",
           w, avg, ms * 1e3 / reps, (double)w * reps / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
