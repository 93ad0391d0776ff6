// small.cu -- the n x n (and s x n) factorizations of the method, replicated work
// that does not scale with m: HouseholderQR of the sketch (only R kept, H never
// formed), Cholesky with breakdown detection, triangular inverse
// for the CholeskyQR2 tail, upper x upper products (R = S U P:282, N = D Y, R = J N
// P:711-717) and the status word.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

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
  note_launch(); status_init_kernel<<<1, 1, 0, st>>>(status);
  return cudaGetLastError();
}
cudaError_t launch_status_finish(const unsigned long long* status, void* info, cudaStream_t st) {
  note_launch(); status_finish_kernel<<<1, 1, 0, st>>>(status, (rlhc_info_t*)info);
  return cudaGetLastError();
}

__global__ void fill_i32_kernel(int* p, int64_t count, int value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) p[i] = value;
}
cudaError_t launch_fill_i32(int* p, int64_t count, int value, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>(ceil_div<int64_t>(count, 256), 4096);
  note_launch(); fill_i32_kernel<<<grid, 256, 0, st>>>(p, count, value);
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
// One CTA of 32 warps.  Per step: warp 0 forms the reflector of column k; barrier;
// warp (j mod 32) applies it to column j (dot product and update, lanes over rows);
// barrier.  The working copy (row stride n+1: conflict-free column access) lives in
// shared memory when it fits, else in `work`.
__global__ void __launch_bounds__(1024)
hqr_kernel(const double* __restrict__ A, int s, int n, int64_t lda, const double* __restrict__ sgn_ref,
           double* __restrict__ S, double* work, int use_smem, unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ double coef[2];  // beta, tau
  __shared__ int flag;
  double* Wm = use_smem ? dsm : work;
  const int ld = n + 1;
  for (int i = warp_id(); i < s; i += 32)
    for (int j = lane_id(); j < n; j += 32) Wm[(int64_t)i * ld + j] = A[(int64_t)i * lda + j];
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  const int lane = lane_id(), wp = warp_id();
  for (int k = 0; k < n; k++) {
    if (wp == 0) {
      double part = 0.0;
      for (int i = k + 1 + lane; i < s; i += 32) { double x = Wm[(int64_t)i * ld + k]; part = __fma_rn(x, x, part); }
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double alpha = Wm[(int64_t)k * ld + k];
      const double xnorm = __dsqrt_rn(part);
      double beta = alpha, tau = 0.0, sc = 0.0;
      if (xnorm != 0.0) {
        beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, xnorm);
        tau = __ddiv_rn(beta - alpha, beta);
        sc = __ddiv_rn(1.0, alpha - beta);
        for (int i = k + 1 + lane; i < s; i += 32) Wm[(int64_t)i * ld + k] *= sc;
      } else if (alpha == 0.0 && lane == 0) {
        report(status, RLHC_ERANKDEF, RLHC_STAGE_HQR, k);
        flag = 1;
      }
      if (lane == 0) { coef[0] = beta; coef[1] = tau; }
    }
    __syncthreads();
    if (flag) break;
    const double tau = coef[1];
    if (tau != 0.0) {
      for (int j = k + 1 + wp; j < n; j += 32) {
        double acc = 0.0;
        for (int i = k + 1 + lane; i < s; i += 32) acc = __fma_rn(Wm[(int64_t)i * ld + k], Wm[(int64_t)i * ld + j], acc);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double tw = tau * (Wm[(int64_t)k * ld + j] + acc);
        __syncwarp();
        if (lane == 0) Wm[(int64_t)k * ld + j] -= tw;
        for (int i = k + 1 + lane; i < s; i += 32)
          Wm[(int64_t)i * ld + j] = __fma_rn(-Wm[(int64_t)i * ld + k], tw, Wm[(int64_t)i * ld + j]);
      }
    }
    if (threadIdx.x == 0) Wm[(int64_t)k * ld + k] = coef[0];
    __syncthreads();
  }
  for (int i = wp; i < n; i += 32) {
    const double d = Wm[(int64_t)i * ld + i];
    const bool flip = sgn_ref && ((d < 0.0) != (sgn_ref[(int64_t)i * n + i] < 0.0));
    for (int j = lane; j < n; j += 32) {
      double v = (j >= i) ? Wm[(int64_t)i * ld + j] : 0.0;
      S[(int64_t)i * n + j] = flip ? -v : v;
    }
  }
}

size_t hqr_ws_bytes(int s, int n) { return ((size_t)s * (n + 1)) * sizeof(double); }

cudaError_t launch_hqr(const double* A, int s, int n, int64_t lda, const double* sgn_ref, double* S, double* work,
                       unsigned long long* status, cudaStream_t st) {
  size_t need = hqr_ws_bytes(s, n);
  int use_smem = need <= 200 * 1024;
  size_t smem = use_smem ? need : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(hqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  note_launch(); hqr_kernel<<<1, 1024, smem, st>>>(A, s, n, lda, sgn_ref, S, work, use_smem, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Cholesky (+ inverse)
// Upper R with R^T R = G, right-looking on a working copy (row stride n+1):
// per step k one thread forms r_kk (a pivot <= 0 or non-finite -> EBREAKDOWN(stage, k),
// SPEC S:55, and the factorization stops), row k is divided by r_kk, and warp (j mod 32)
// updates column j.  With Rinv != NULL the kernel then inverts R (thread per column,
// back substitution in shared memory) for the CholeskyQR2 tail.
__global__ void __launch_bounds__(1024)
chol_kernel(const double* __restrict__ G, int n, double* __restrict__ R, double* __restrict__ Rinv, double* work,
            int use_smem, int stage, unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ int flag;
  __shared__ double rkk_s;
  const int ld = n + 1;
  double* C = use_smem ? dsm : work;
  double* Xi = C + (size_t)n * ld;  // inverse workspace (smem when it fits)
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    C[i * ld + j] = G[idx];
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  const int lane = lane_id(), wp = warp_id();
  for (int k = 0; k < n; k++) {
    if (threadIdx.x == 0) {
      double d = C[k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) { report(status, RLHC_EBREAKDOWN, stage, k); flag = 1; }
      else { rkk_s = __dsqrt_rn(d); C[k * ld + k] = rkk_s; }
    }
    __syncthreads();
    if (flag) break;
    const double rkk = rkk_s;
    for (int j = k + 1 + threadIdx.x; j < n; j += blockDim.x) C[k * ld + j] = __ddiv_rn(C[k * ld + j], rkk);
    __syncthreads();
    for (int j = k + 1 + wp; j < n; j += 32) {
      const double ckj = C[k * ld + j];
      for (int i = k + 1 + lane; i <= j; i += 32) C[i * ld + j] = __fma_rn(-C[k * ld + i], ckj, C[i * ld + j]);
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx - i * n;
    R[idx] = (j >= i) ? C[i * ld + j] : 0.0;
  }
  if (Rinv && !flag) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      for (int i = j; i >= 0; i--) {
        double sum = (i == j) ? 1.0 : 0.0;
        for (int l = i + 1; l <= j; l++) sum = __fma_rn(-C[i * ld + l], Xi[l * ld + j], sum);
        Xi[i * ld + j] = __ddiv_rn(sum, C[i * ld + i]);
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      int i = idx / n, j = idx - i * n;
      Rinv[idx] = (j >= i) ? Xi[i * ld + j] : 0.0;
    }
  }
}

size_t chol_ws_bytes(int n) { return 2 * (size_t)n * (n + 1) * sizeof(double); }

cudaError_t launch_chol(const double* G, int n, double* R, double* work, int stage, unsigned long long* status,
                        cudaStream_t st) {
  return launch_chol_inv(G, n, R, nullptr, work, stage, status, st);
}

cudaError_t launch_chol_inv(const double* G, int n, double* R, double* Rinv, double* work, int stage,
                            unsigned long long* status, cudaStream_t st) {
  size_t need = chol_ws_bytes(n);
  int use_smem = need <= 200 * 1024;
  if (!use_smem && !work) return cudaErrorInvalidValue;
  size_t smem = use_smem ? need : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
  }
  note_launch(); chol_kernel<<<1, 1024, smem, st>>>(G, n, R, Rinv, work, use_smem, stage, status);
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
  note_launch(); tri_inv_kernel<<<ceil_div(n, 64), 64, 0, st>>>(T, n, Tinv);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ upper x upper
// C = A B for upper-triangular A, B stored with exact zeros below the diagonal: a
// shared-memory tiled product (16 x 16 tiles, k ascending); the zero parts contribute
// exact zeros, so C's strict lower part is exactly 0 and its upper part is
// sum_{k=i..j} A_ik B_kj.  Tiles entirely below the diagonal are written as zeros.
__global__ void __launch_bounds__(256) trmm_uu_kernel(const double* __restrict__ A, const double* __restrict__ B, int n,
                                                      double* __restrict__ C) {
  __shared__ double As[16][17], Bs[16][17];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  double acc = 0.0;
  if (blockIdx.y <= blockIdx.x) {
    for (int k0 = blockIdx.y * 16; k0 <= (int)blockIdx.x * 16 && k0 < n; k0 += 16) {
      As[ty][tx] = (i < n && k0 + tx < n) ? A[(int64_t)i * n + k0 + tx] : 0.0;
      Bs[ty][tx] = (k0 + ty < n && j < n) ? B[(int64_t)(k0 + ty) * n + j] : 0.0;
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; kk++) acc = __fma_rn(As[ty][kk], Bs[kk][tx], acc);
      __syncthreads();
    }
  }
  if (i < n && j < n) C[(int64_t)i * n + j] = (j >= i) ? acc : 0.0;
}
cudaError_t launch_trmm_uu(const double* A, const double* B, int n, double* C, cudaStream_t st) {
  dim3 grid(ceil_div(n, 16), ceil_div(n, 16));
  note_launch(); trmm_uu_kernel<<<grid, 256, 0, st>>>(A, B, n, C);
  return cudaGetLastError();
}

}  // namespace rlhc
