// Dependent-chain latencies (cycles) of the ops on the tournament select's critical path.
#include <cstdio>
__global__ void lat(long long* out, int n, int seed) {
  const int lane = threadIdx.x & 31;
  int v = lane * 7 + seed;
  unsigned u = lane * 13u + seed;
  double d = 1.0 + lane * 1e-3 * seed;
  long long t0, t1;
  // redux.max chain
  t0 = clock64();
  for (int i = 0; i < n; i++) v = __reduce_max_sync(0xffffffffu, v) - lane;
  t1 = clock64(); out[0] = (t1 - t0) / n;
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < n; i++) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) + 1;
  t1 = clock64(); out[1] = (t1 - t0) / n;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; i++) d = __fma_rn(d, 0.999, 1e-3);
  t1 = clock64(); out[2] = (t1 - t0) / n;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; i++) d = __dmul_rn(d, 1.0000001);
  t1 = clock64(); out[3] = (t1 - t0) / n;
  // ballot chain
  t0 = clock64();
  for (int i = 0; i < n; i++) u = __ballot_sync(0xffffffffu, (u >> (lane & 7)) & 1) + lane;
  t1 = clock64(); out[4] = (t1 - t0) / n;
  // double hi-word extraction + int op chain
  t0 = clock64();
  for (int i = 0; i < n; i++) { int h = __double2hiint(d) & 0x7fffffff; d = __hiloint2double(h ^ (i & 1), __double2loint(d)); }
  t1 = clock64(); out[5] = (t1 - t0) / n;
  // redux.min unsigned
  t0 = clock64();
  for (int i = 0; i < n; i++) u = __reduce_min_sync(0xffffffffu, u) + lane;
  t1 = clock64(); out[6] = (t1 - t0) / n;
  if (v == 12345 && u == 7 && d == 0.5) out[7] = 1;
}
int main() {
  long long* o; cudaMallocManaged(&o, 64);
  lat<<<1, 32>>>(o, 10, 1); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, 1000, 1); cudaDeviceSynchronize();
  printf("{\"redux_max\":%lld,\"shfl\":%lld,\"dfma\":%lld,\"dmul\":%lld,\"ballot\":%lld,\"hi_extract_roundtrip\":%lld,\"redux_min\":%lld}\n",
         o[0], o[1], o[2], o[3], o[4], o[5], o[6]);
  return 0;
}
