// Probe: phase timeline of rowsolve_kernel (CTA 0, warp 0) at cfg2's shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DRLHC_RS_TRACE \
//      -o prs prs.cu ../../paper_2412_06551_b200/csrc/small.cu
#include <cstdio>
#include <vector>
#include "../../paper_2412_06551_b200/csrc/rows.cu"
using namespace rlhc;
int main(int argc, char** argv) {
  const int64_t m = 65536;
  const int n = 64;
  const int gram = argc > 1 ? atoi(argv[1]) : 1;
  std::vector<double> hT(n * n, 0.0), hA(m * n);
  for (int i = 0; i < n; i++)
    for (int j = i; j < n; j++) hT[i * n + j] = (i == j) ? 1.0 + 0.01 * i : 0.001 * (i + j);
  for (int64_t i = 0; i < m * n; i++) hA[i] = 1e-3 * (double)((i * 7919) % 1000);
  std::vector<double> hr(n);
  for (int i = 0; i < n; i++) hr[i] = 1.0 / hT[i * n + i];
  double *A, *T, *rd, *out, *part, *G;
  cudaMalloc(&A, m * n * 8); cudaMalloc(&T, n * n * 8); cudaMalloc(&rd, n * 8); cudaMalloc(&out, m * n * 8);
  cudaMalloc(&part, rowsolve_partials_bytes(m, n)); cudaMalloc(&G, n * n * 8);
  cudaMemcpy(A, hA.data(), m * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(T, hT.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(rd, hr.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; it++) {
    cudaEventRecord(e0);
    launch_rowsolve(A, n, m, n, T, rd, out, n, nullptr, nullptr, part, gram ? G : nullptr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long t[256];
  cudaMemcpyFromSymbol(t, g_rs_trace, sizeof(t));
  printf("err %s  kernel(s) %.1f us\n", cudaGetErrorString(cudaGetLastError()), ms * 1000);
  for (int i = 1; i < 12; i++) if (t[i] > t[0]) printf("  trace %d: +%lld cycles\n", i, t[i] - t[0]);
}
