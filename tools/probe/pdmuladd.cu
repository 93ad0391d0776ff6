// FP64-pipe throughput of the oracle-order term acc = RN(acc - RN(w * y)) (a DMUL + a DADD),
// against DFMA, register-resident, vs warps per SM and independent accumulators per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, bool FMA>
__global__ void tput(double* out, int iters) {
  // distinct y per accumulator: no product can be shared between terms (an earlier version
  // reused w * y across accumulators and measured only the DADDs)
  double acc[CH], ys[CH];
  for (int i = 0; i < CH; i++) acc[i] = threadIdx.x * 1e-3 + i, ys[i] = 1.0 + threadIdx.x * 1e-7 + i * 1e-5;
  double w = 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      const double y = ys[i];
      if (FMA) acc[i] = __fma_rn(-w, y, acc[i]);
      else acc[i] = __dsub_rn(acc[i], __dmul_rn(w, y));
    }
    w = __dadd_rn(w, 1e-30);
  }
  double s = 0;
  for (int i = 0; i < CH; i++) s += acc[i];
  if (s == 12345.0) out[0] = s;
}
template <int CH, bool FMA>
void run(int wps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, 8);
  const int iters = 4000, thr = 32 * wps;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  tput<CH, FMA><<<sms, thr>>>(o, 10);
  cudaEventRecord(a);
  tput<CH, FMA><<<sms, thr>>>(o, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double terms = (double)sms * thr * iters * CH;
  printf("{\"op\":\"%s\",\"warps_per_sm\":%d,\"chains\":%d,\"Gterms_per_s\":%.1f,\"fp64_instr_T_per_s\":%.2f}\n",
         FMA ? "dfma" : "dmul+dadd", wps, CH, terms / ms / 1e6, terms * (FMA ? 1 : 2) / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int wps : {4, 8, 16}) {
    run<16, false>(wps); run<32, false>(wps); run<32, true>(wps);
  }
  return 0;
}
