// Probe: latency of warp collectives on sm_100a (dependent chains, one warp).
#include <cstdio>
__global__ void k(int* out, long long* t, int seed) {
  int v = threadIdx.x ^ seed;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; i++) v = __reduce_max_sync(0xffffffffu, v) + threadIdx.x;
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; i++) v = __shfl_sync(0xffffffffu, v, (v & 31)) + 1;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; i++) v = (int)__ballot_sync(0xffffffffu, (v & 1)) + threadIdx.x;
  long long t3 = clock64();
  double d = v * 1.5;
#pragma unroll 1
  for (int i = 0; i < 100; i++) d = __drcp_rn(d + 1.0);
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; i++) d = __fma_rn(d, d, 1.0);
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; i++) v = __reduce_min_sync(0xffffffffu, v) ^ threadIdx.x;
  long long t6 = clock64();
  out[threadIdx.x] = v + (int)d;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; }
}
int main() {
  int* o; long long* t; cudaMalloc(&o, 128); cudaMalloc(&t, 64);
  for (int r = 0; r < 3; r++) k<<<1, 32>>>(o, t, r);
  long long h[6]; cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
  printf("per-iteration cycles (incl. loop + 1 dependent ALU op): redux.max %.1f shfl %.1f ballot %.1f drcp+dadd %.1f dfma %.1f redux.min %.1f\n",
         h[0] / 100., h[1] / 100., h[2] / 100., h[3] / 100., h[4] / 100., h[5] / 100.);
}
