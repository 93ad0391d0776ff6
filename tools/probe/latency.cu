// Throwaway probe: per-iteration latency of single-CTA serial primitives on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_sync(int it, double* out) {
  double v = threadIdx.x;
  for (int i = 0; i < it; i++) { __syncthreads(); v += 1.0; }
  if (v == -1) out[0] = v;
}
__global__ void k_redux(int it, double* out) {
  int v = threadIdx.x;
  for (int i = 0; i < it; i++) v = __reduce_max_sync(0xffffffffu, v) + 1;
  if (v == -1) out[0] = v;
}
__global__ void k_shfl(int it, double* out) {
  double v = threadIdx.x;
  for (int i = 0; i < it; i++) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.0;
  if (v == -1) out[0] = v;
}
__global__ void k_ddiv(int it, double* out) {
  double v = threadIdx.x + 1.5;
  for (int i = 0; i < it; i++) v = __ddiv_rn(1.0, v) + 1.5;
  if (v == -1) out[0] = v;
}
__global__ void k_drcp(int it, double* out) {
  double v = threadIdx.x + 1.5;
  for (int i = 0; i < it; i++) v = __drcp_rn(v) + 1.5;
  if (v == -1) out[0] = v;
}
__global__ void k_dsqrt(int it, double* out) {
  double v = threadIdx.x + 1.5;
  for (int i = 0; i < it; i++) v = __dsqrt_rn(v * 3.0 + 0.25) + 1.5;
  if (v == -1) out[0] = v;
}
__global__ void k_dfma(int it, double* out) {
  double v = threadIdx.x + 1.5;
  for (int i = 0; i < it; i++) v = __fma_rn(v, 0.999, 1e-3);
  if (v == -1) out[0] = v;
}
__global__ void k_smem(int it, double* out) {
  __shared__ double s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  int idx = threadIdx.x;
  double v = 0;
  for (int i = 0; i < it; i++) { v += s[idx]; idx = ((int)v + i) & 1023; }
  if (v == -1) out[0] = v;
}
__global__ void k_syncshared(int it, double* out) {  // publish + sync + read (producer/consumer step)
  __shared__ double s[2];
  double v = threadIdx.x;
  for (int i = 0; i < it; i++) {
    if (threadIdx.x == 0) s[i & 1] = v;
    __syncthreads();
    v = s[i & 1] + 1.0;
  }
  if (v == -1) out[0] = v;
}

__global__ void k_sqrt_std(int it, double* out) {
  double v = threadIdx.x + 1.5;
  for (int i = 0; i < it; i++) v = sqrt(v * 3.0 + 0.25) + 1.5;
  if (v == -1) out[0] = v;
}
__global__ void k_smem_rw(int it, double* out) {  // dependent smem store->load round trips
  __shared__ double s[64];
  double v = threadIdx.x;
  for (int i = 0; i < it; i++) { s[threadIdx.x & 63] = v; __syncwarp(); v = s[(threadIdx.x + 1) & 63] + 1.0; __syncwarp(); }
  if (v == -1) out[0] = v;
}
__global__ void k_dmma_chain(int it, double* out) {
  double c0 = threadIdx.x, c1 = 1.0, a = 0.5, b = 0.25;
  for (int i = 0; i < it; i++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  if (c0 == -1) out[0] = c0 + c1;
}
__global__ void k_dmma_4chains(int it, double* out) {
  double c[4][2] = {{1, 1}, {2, 2}, {3, 3}, {4, 4}};
  double a = 0.5, b = 0.25;
  for (int i = 0; i < it; i++)
#pragma unroll
    for (int q = 0; q < 4; q++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  if (c[0][0] == -1) out[0] = c[1][0] + c[2][0] + c[3][0];
}
__global__ void k_ldg_chain(int it, double* out) {
  __shared__ int dummy;
  const double* p = out + 8;
  int idx = threadIdx.x;
  double v = 0;
  for (int i = 0; i < it; i++) { v += p[idx]; idx = ((int)v + i) & 255; }
  if (v == -1) dummy = 1, out[0] = v;
}

template <typename F>
void run(const char* name, F f, int threads) {
  double* o; cudaMalloc(&o, 8 * 512); cudaMemset(o, 0, 8 * 512);
  int it = 20000;
  f<<<1, threads>>>(100, o);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); f<<<1, threads>>>(it, o); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-14s threads=%4d  %7.1f ns/iter  (%6.0f cycles @ max clock)\n", name, threads, ms * 1e6 / it,
         ms * 1e6 / it * clk / 1e6);
}

int main() {
  for (int th : {32, 256, 1024}) {
    run("syncthreads", k_sync, th);
    run("sync+smem", k_syncshared, th);
  }
  run("redux", k_redux, 32);
  run("shfl.f64", k_shfl, 32);
  run("ddiv_rn", k_ddiv, 32);
  run("drcp_rn", k_drcp, 32);
  run("dsqrt_rn", k_dsqrt, 32);
  run("dfma", k_dfma, 32);
  run("lds chase", k_smem, 32);
  run("sqrt()", k_sqrt_std, 32);
  run("smem st/ld rt", k_smem_rw, 32);
  run("dmma chain", k_dmma_chain, 32);
  run("dmma 4chains", k_dmma_4chains, 32);
  run("dmma chain", k_dmma_chain, 256);
  run("ldg chase L1", k_ldg_chain, 32);
  return 0;
}
