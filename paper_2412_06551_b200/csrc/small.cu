// small.cu -- the n x n (and s x n) factorizations of the method, replicated work
// that does not scale with m: HouseholderQR of the sketch (only R kept, H never
// formed), Cholesky with breakdown detection, triangular inverse
// for the CholeskyQR2 tail, upper x upper products (R = S U P:282, N = D Y, R = J N
// P:711-717) and the status word.
#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

// ------------------------------------------------------------------ status
__global__ void status_init_kernel(unsigned long long* status) { *status = kStatusOK; }
__global__ void status_finish_kernel(const unsigned long long* status, rlhc_info_t* info) {
  unsigned long long k = *status;
  if (k == kStatusOK) {
    info->code = RLHC_OK; info->stage = 0; info->index = 0;
  } else {
    info->stage = (int32_t)(k >> 56);
    info->code = (int32_t)((k >> 48) & 0xff);
    info->index = (int64_t)(k & 0xFFFFFFFFFFFFull);
  }
}
cudaError_t launch_status_init(unsigned long long* status, cudaStream_t st) {
  status_init_kernel<<<1, 1, 0, st>>>(status);
  return cudaGetLastError();
}
cudaError_t launch_status_finish(const unsigned long long* status, void* info, cudaStream_t st) {
  status_finish_kernel<<<1, 1, 0, st>>>(status, (rlhc_info_t*)info);
  return cudaGetLastError();
}

__global__ void fill_i32_kernel(int* p, int64_t count, int value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) p[i] = value;
}
cudaError_t launch_fill_i32(int* p, int64_t count, int value, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(ceil_div<int64_t>(count, 256), 4096);
  fill_i32_kernel<<<grid, 256, 0, st>>>(p, count, value);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ block reduce
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int nw = blockDim.x >> 5;
  __syncthreads();
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < nw; q++) s += red[q];  // fixed order, every thread the same
  return s;
}

// ------------------------------------------------------------------ Householder R
// LAPACK dgeqr2 order (DESIGN.md R#O7): beta = -sign(alpha) ||x||, tau = (beta -
// alpha)/beta, v = x(2:)/(alpha - beta); A(k:, k+1:) -= tau v (v^T A(k:, k+1:)).
// One CTA; the working copy lives in shared memory when it fits, else in `work`.
__global__ void __launch_bounds__(1024)
hqr_kernel(const double* __restrict__ A, int s, int n, int64_t lda, const double* __restrict__ sgn_ref,
           double* __restrict__ S, double* work, int use_smem, unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ double red[32];
  __shared__ double coef[3];  // beta, tau, scale
  __shared__ int flag;
  double* Wm = use_smem ? dsm : work;
  double* tw = use_smem ? (dsm + (size_t)s * n) : (work + (size_t)s * n);
  for (int64_t idx = threadIdx.x; idx < (int64_t)s * n; idx += blockDim.x) {
    int i = (int)(idx / n), j = (int)(idx - (int64_t)i * n);
    Wm[idx] = A[(int64_t)i * lda + j];
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  const int lane = lane_id(), wp = warp_id(), nw = blockDim.x >> 5;
  for (int k = 0; k < n; k++) {
    double part = 0.0;
    for (int i = k + 1 + threadIdx.x; i < s; i += blockDim.x) { double x = Wm[(int64_t)i * n + k]; part = __fma_rn(x, x, part); }
    double xn2 = block_sum(part, red);
    if (threadIdx.x == 0) {
      double alpha = Wm[(int64_t)k * n + k];
      double xnorm = __dsqrt_rn(xn2);
      if (xnorm == 0.0 && alpha == 0.0) { report(status, RLHC_ERANKDEF, RLHC_STAGE_HQR, k); flag = 1; }
      if (xnorm == 0.0) { coef[0] = alpha; coef[1] = 0.0; coef[2] = 0.0; }
      else {
        double beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, xnorm);
        coef[0] = beta;
        coef[1] = __ddiv_rn(beta - alpha, beta);
        coef[2] = __ddiv_rn(1.0, alpha - beta);
      }
    }
    __syncthreads();
    if (flag) break;
    const double tau = coef[1];
    if (tau != 0.0) {
      const double sc = coef[2];
      for (int i = k + 1 + threadIdx.x; i < s; i += blockDim.x) Wm[(int64_t)i * n + k] *= sc;
      __syncthreads();
      if (threadIdx.x == 0) Wm[(int64_t)k * n + k] = coef[0];
      // w_j = A[k][j] + sum_i v_i A[i][j]   (warp per column, lanes over rows)
      for (int j = k + 1 + wp; j < n; j += nw) {
        double acc = 0.0;
        for (int i = k + 1 + lane; i < s; i += 32) acc = __fma_rn(Wm[(int64_t)i * n + k], Wm[(int64_t)i * n + j], acc);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) tw[j] = tau * (Wm[(int64_t)k * n + j] + acc);
      }
      __syncthreads();
      const int nc = n - k - 1;
      for (int64_t idx = threadIdx.x; idx < (int64_t)(s - k) * nc; idx += blockDim.x) {
        int i = k + (int)(idx / nc), j = k + 1 + (int)(idx % nc);
        double v = (i == k) ? 1.0 : Wm[(int64_t)i * n + k];
        Wm[(int64_t)i * n + j] = __fma_rn(-v, tw[j], Wm[(int64_t)i * n + j]);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    double v = (j >= i) ? Wm[(int64_t)i * n + j] : 0.0;
    if (sgn_ref) {
      double d = Wm[(int64_t)i * n + i], ref = sgn_ref[(int64_t)i * n + i];
      if ((d < 0.0) != (ref < 0.0)) v = -v;
    }
    S[idx] = v;
  }
}

size_t hqr_ws_bytes(int s, int n) { return ((size_t)s * n + n) * sizeof(double); }

cudaError_t launch_hqr(const double* A, int s, int n, int64_t lda, const double* sgn_ref, double* S, double* work,
                       unsigned long long* status, cudaStream_t st) {
  size_t need = hqr_ws_bytes(s, n);
  int use_smem = need <= 200 * 1024;
  size_t smem = use_smem ? need : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(hqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  hqr_kernel<<<1, 1024, smem, st>>>(A, s, n, lda, sgn_ref, S, work, use_smem, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Cholesky
// Upper R with R^T R = G, right-looking on a working copy; a pivot <= 0 or
// non-finite -> EBREAKDOWN(stage, k) and the factorization stops.
__global__ void __launch_bounds__(1024)
chol_kernel(const double* __restrict__ G, int n, double* __restrict__ R, double* work, int use_smem, int stage,
            unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ int flag;
  __shared__ double rkk_s;
  double* C = use_smem ? dsm : work;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) C[idx] = G[idx];
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int k = 0; k < n; k++) {
    if (threadIdx.x == 0) {
      double d = C[(int64_t)k * n + k];
      if (!(d > 0.0) || !isfinite(d)) { report(status, RLHC_EBREAKDOWN, stage, k); flag = 1; }
      else { rkk_s = __dsqrt_rn(d); C[(int64_t)k * n + k] = rkk_s; }
    }
    __syncthreads();
    if (flag) break;
    const double rkk = rkk_s;
    for (int j = k + 1 + threadIdx.x; j < n; j += blockDim.x) C[(int64_t)k * n + j] = __ddiv_rn(C[(int64_t)k * n + j], rkk);
    __syncthreads();
    const int nc = n - k - 1;
    for (int64_t idx = threadIdx.x; idx < (int64_t)nc * nc; idx += blockDim.x) {
      int i = k + 1 + (int)(idx / nc), j = k + 1 + (int)(idx % nc);
      if (j >= i) C[(int64_t)i * n + j] = __fma_rn(-C[(int64_t)k * n + i], C[(int64_t)k * n + j], C[(int64_t)i * n + j]);
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    R[idx] = (j >= i) ? C[idx] : 0.0;
  }
}

cudaError_t launch_chol(const double* G, int n, double* R, double* work, int stage, unsigned long long* status,
                        cudaStream_t st) {
  size_t need = (size_t)n * n * sizeof(double);
  int use_smem = need <= 200 * 1024;
  size_t smem = use_smem ? need : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  chol_kernel<<<1, 1024, smem, st>>>(G, n, R, work, use_smem, stage, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ T^{-1}
// Upper-triangular inverse, one thread per column (back substitution), zero lower part.
__global__ void tri_inv_kernel(const double* __restrict__ T, int n, double* __restrict__ Ti) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = n - 1; i > j; i--) Ti[(int64_t)i * n + j] = 0.0;
  Ti[(int64_t)j * n + j] = __ddiv_rn(1.0, T[(int64_t)j * n + j]);
  for (int i = j - 1; i >= 0; i--) {
    double s = 0.0;
    for (int l = i + 1; l <= j; l++) s = __fma_rn(T[(int64_t)i * n + l], Ti[(int64_t)l * n + j], s);
    Ti[(int64_t)i * n + j] = __ddiv_rn(-s, T[(int64_t)i * n + i]);
  }
}
cudaError_t launch_tri_inv(const double* T, int n, double* Tinv, cudaStream_t st) {
  tri_inv_kernel<<<ceil_div(n, 64), 64, 0, st>>>(T, n, Tinv);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ upper x upper
__global__ void trmm_uu_kernel(const double* __restrict__ A, const double* __restrict__ B, int n, double* __restrict__ C) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
  double acc = 0.0;
  if (j >= i)
    for (int k = i; k <= j; k++) acc = __fma_rn(A[(int64_t)i * n + k], B[(int64_t)k * n + j], acc);
  C[e] = acc;
}
cudaError_t launch_trmm_uu(const double* A, const double* B, int n, double* C, cudaStream_t st) {
  int64_t total = (int64_t)n * n;
  trmm_uu_kernel<<<(int)ceil_div<int64_t>(total, 256), 256, 0, st>>>(A, B, n, C);
  return cudaGetLastError();
}

}  // namespace rlhc
