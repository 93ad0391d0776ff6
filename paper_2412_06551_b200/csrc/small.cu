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

// ------------------------------------------------------------------ T^{-1}
// Upper-triangular inverse (for D^-1 and J^-1 of the CholeskyQR passes, kappa <= ~7): one
// warp per column j of T^-1, back substitution x_i = (delta_ij - sum_{l=i+1..j} T_il x_l)/T_ii
// for i = j .. 0 with x in shared memory; each dot product is split over the lanes
// (fixed lane partition, fixed butterfly) -- deterministic.  The zero lower part is written.
constexpr int TI_WARPS = 4;
__global__ void __launch_bounds__(32 * TI_WARPS) tri_inv_kernel(const double* __restrict__ T, int n,
                                                                double* __restrict__ Ti) {
  extern __shared__ double ti_x[];  // [TI_WARPS][n]
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int j = blockIdx.x * TI_WARPS + wq;
  if (j >= n) return;
  double* x = ti_x + (size_t)wq * n;
  for (int i = j + 1 + lane; i < n; i += 32) Ti[(int64_t)i * n + j] = 0.0;
  for (int i = j; i >= 0; i--) {
    const double* Tr = T + (int64_t)i * n;
    double s = 0.0;
    for (int l = i + 1 + lane; l <= j; l += 32) s = __fma_rn(Tr[l], x[l], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double xi = __ddiv_rn((i == j ? 1.0 : 0.0) - s, Tr[i]);
    if (lane == 0) x[i] = xi;
    __syncwarp();
    if (lane == 0) Ti[(int64_t)i * n + j] = xi;
  }
}
cudaError_t launch_tri_inv(const double* T, int n, double* Tinv, cudaStream_t st) {
  const size_t smem = (size_t)TI_WARPS * n * sizeof(double);
  static DevFlags attr;
  if (smem > 48 * 1024)
    if (cudaError_t e = smem_attr(attr, tri_inv_kernel, (int)smem)) return e;
  note_launch();
  tri_inv_kernel<<<ceil_div(n, TI_WARPS), 32 * TI_WARPS, smem, st>>>(T, n, Tinv);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ comparison-method helpers
// SCholeskyQR shift (R#21): G += s I with s = 11 (m n u + (n + 1) u) max_k G_kk
// (||X||_g^2 = the largest squared column norm = the largest diagonal entry of X^T X).
__global__ void shift_diag_kernel(double* G, int n, int64_t m) {
  __shared__ double red[32];
  double g = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) g = fmax(g, G[(int64_t)k * n + k]);
  for (int o = 16; o; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g;
  __syncthreads();
  if (threadIdx.x < 32) {
    g = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (threadIdx.x == 0) red[0] = g;
  }
  __syncthreads();
  const double u = 0x1p-53;
  const double shift = 11.0 * ((double)m * (double)n * u + (double)(n + 1) * u) * red[0];
  for (int k = threadIdx.x; k < n; k += blockDim.x) G[(int64_t)k * n + k] += shift;
}
cudaError_t launch_shift_diag(double* G, int n, int64_t m, cudaStream_t st) {
  note_launch(); shift_diag_kernel<<<1, 256, 0, st>>>(G, n, m);
  return cudaGetLastError();
}

// rows of the upper-triangular T with a negative diagonal negated (diag(T) > 0)
__global__ void flip_neg_rows_kernel(double* T, int n) {
  const int k = blockIdx.x;
  const bool neg = T[(int64_t)k * n + k] < 0.0;
  if (neg)
    for (int j = threadIdx.x; j < n; j += blockDim.x) T[(int64_t)k * n + j] = -T[(int64_t)k * n + j];
}
cudaError_t launch_flip_neg_rows(double* T, int n, cudaStream_t st) {
  note_launch(); flip_neg_rows_kernel<<<n, 128, 0, st>>>(T, n);
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
