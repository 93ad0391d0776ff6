// DMMA m8n8k4.f64 throughput vs warps per SM and independent chains per warp
// (register-resident operands), and with fragments loaded from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dmma_tput(double* out, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; i++) { c[i][0] = 0; c[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < CH; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
// 4x4 fragment tile per warp, fragments from shared memory each k-step (like a GEMM mainloop)
__global__ void dmma_smem(double* out, int iters) {
  __shared__ double A[1][128][20];
  __shared__ double B[1][16][68];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < 1 * 128 * 20; i += blockDim.x) (&A[0][0][0])[i] = i * 1e-6;
  for (int i = threadIdx.x; i < 1 * 16 * 68; i += blockDim.x) (&B[0][0][0])[i] = i * 1e-6;
  __syncthreads();
  const int wi = ((wp >> 1) & 3) * 32, wj = (wp & 1) * 32, st = 0;
  double acc[4][4][2] = {};
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = A[st][wi + a * 8 + g][k0 + t];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = B[st][k0 + t][wj + b * 8 + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[a][b][0]), "+d"(acc[a][b][1]) : "d"(af[a]), "d"(bf[b]));
    }
  }
  double s = 0;
  for (int a = 0; a < 4; a++) for (int b = 0; b < 4; b++) s += acc[a][b][0] + acc[a][b][1];
  if (s == 12345.0) out[0] = s;
}
template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  const int IT = 4096;
  const int sms = 148;
  for (int wps : {4, 8, 16, 32, 64}) {  // warps per SM
    int warps_per_block = wps < 16 ? wps : 16, blocks = sms * (wps / warps_per_block);
    for (int ch : {4, 8, 16, 32}) {
      float ms;
      if (ch == 4) ms = timeit([&] { dmma_tput<4><<<blocks, 32 * warps_per_block>>>(out, IT * 8); });
      else if (ch == 8) ms = timeit([&] { dmma_tput<8><<<blocks, 32 * warps_per_block>>>(out, IT * 4); });
      else if (ch == 16) ms = timeit([&] { dmma_tput<16><<<blocks, 32 * warps_per_block>>>(out, IT * 2); });
      else ms = timeit([&] { dmma_tput<32><<<blocks, 32 * warps_per_block>>>(out, IT); });
      double fl = 2.0 * blocks * warps_per_block * 32.0 * IT * 256;
      printf("{\"warps_per_sm\":%d,\"chains\":%d,\"tflops\":%.2f}\n", wps, ch, fl / ms / 1e9);
    }
  }
  for (int wpb : {8, 16}) {
    for (int bps : {1, 2, 3, 4}) {
      if (wpb * bps > 32) continue;
      int blocks = sms * bps;
      float ms = timeit([&] { dmma_smem<<<blocks, 32 * wpb>>>(out, 2048); });
      double fl = 2.0 * blocks * wpb * 2048.0 * 4 * 16 * 256;
      printf("{\"smem_frag\":1,\"warps_per_block\":%d,\"blocks_per_sm\":%d,\"tflops\":%.2f}\n", wpb, bps, fl / ms / 1e9);
    }
  }
  return 0;
}
