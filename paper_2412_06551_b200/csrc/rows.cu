// rows.cu -- m-row streaming kernels: finiteness check, row-wise triangular solve
// X T^{-1} by substitution (R#9), row block times upper-triangular matrix
// (CholeskyQR2 tail with D^{-1}, J^{-1}), and the tall-skinny Gram A^T A.
// Off-diagonal work runs on the FP64 tensor cores (DMMA m8n8k4): measured bitwise equal
// to the fma chain in increasing k, so the substitution reproduces the oracle's
// definition bit for bit (DESIGN.md R#O5).
#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

// ------------------------------------------------------------------ finiteness
__global__ void check_finite_kernel(const double* __restrict__ X, int64_t rows, int n, int64_t ldx,
                                    unsigned long long* status) {
  const int64_t total = rows * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / n;
    int j = (int)(e - i * n);
    double v = X[i * ldx + j];
    if (!isfinite(v)) report(status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, e);
  }
}

cudaError_t launch_check_finite(const double* X, int64_t rows, int n, int64_t ldx, unsigned long long* status,
                                cudaStream_t st) {
  int64_t total = rows * n;
  int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), kSMs * 8);
  if (grid < 1) grid = 1;
  check_finite_kernel<<<grid, 256, 0, st>>>(X, rows, n, ldx, status);
  return cudaGetLastError();
}

// rdiag[k] = 1 / T[k][k] (IEEE), zero or non-finite diagonal -> ESINGULAR(stage, k)
__global__ void rdiag_kernel(const double* __restrict__ T, int n, int64_t ldt, double* __restrict__ rdiag, int stage,
                             unsigned long long* status) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double d = T[(int64_t)k * ldt + k];
    if (d == 0.0 || !isfinite(d)) report(status, RLHC_ESINGULAR, stage, k);
    rdiag[k] = __ddiv_rn(1.0, d);
  }
}

cudaError_t launch_rdiag(const double* T, int n, int64_t ldt, double* rdiag, int stage, unsigned long long* status,
                         cudaStream_t st) {
  rdiag_kernel<<<ceil_div(n, 256), 256, 0, st>>>(T, n, ldt, rdiag, stage, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ substitution
// One warp owns 16 rows (two m8 fragments) of the CTA's row tile, kept in shared
// memory.  Column block jb (8 columns): acc = tile[:, jb] then the chain over the
// already-substituted columns k < min(8 jb, nsub) on DMMA (A = -l, B = T[k, jb]);
// then, inside the 8-wide diagonal block, 16 lanes substitute their rows sequentially:
//   l_k = acc_k * rdiag_k ; acc_j = fma(-l_k, T[k][j], acc_j) for j > k.
template <int NWARP>
__global__ void __launch_bounds__(32 * NWARP)
trsm_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int ncols, int nsub,
                 const double* __restrict__ T, int64_t ldt, const double* __restrict__ rdiag, double* out,
                 int64_t ldo, const int* __restrict__ pivpos, const double* __restrict__ L11, int64_t ldl11) {
  extern __shared__ double S[];
  constexpr int TR = 16 * NWARP;
  const int ncp = (ncols + 7) & ~7;
  const int lds = ncp + 4;
  const int64_t rbase = (int64_t)blockIdx.x * TR;
  for (int idx = threadIdx.x; idx < TR * ncp; idx += blockDim.x) {
    int r = idx / ncp, c = idx - r * ncp;
    int64_t gr = rbase + r;
    S[r * lds + c] = (gr < rows && c < ncols) ? A[gr * lda + c] : 0.0;
  }
  __syncthreads();
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  double* Sw = S + (w * 16) * lds;
  for (int j0 = 0; j0 < ncp; j0 += 8) {
    double acc[2][2];
#pragma unroll
    for (int mf = 0; mf < 2; mf++) {
      acc[mf][0] = Sw[(mf * 8 + g) * lds + j0 + 2 * t];
      acc[mf][1] = Sw[(mf * 8 + g) * lds + j0 + 2 * t + 1];
    }
    const int kend = min(j0, nsub);
    const bool colok = (j0 + g) < ncols;
    for (int k0 = 0; k0 < kend; k0 += 4) {
      const int k = k0 + t;
      double b = (k < kend && colok) ? T[(int64_t)k * ldt + j0 + g] : 0.0;
#pragma unroll
      for (int mf = 0; mf < 2; mf++) {
        double a = (k < kend) ? -Sw[(mf * 8 + g) * lds + k] : 0.0;
        dmma(acc[mf][0], acc[mf][1], a, b);
      }
    }
#pragma unroll
    for (int mf = 0; mf < 2; mf++) {
      Sw[(mf * 8 + g) * lds + j0 + 2 * t] = acc[mf][0];
      Sw[(mf * 8 + g) * lds + j0 + 2 * t + 1] = acc[mf][1];
    }
    __syncwarp();
    if (j0 < nsub && lane < 16) {
      double* row = Sw + lane * lds + j0;
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; q++) v[q] = row[q];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) {
        const int k = j0 + kk;
        if (k < nsub) {
          double l = __dmul_rn(v[kk], rdiag[k]);
          v[kk] = l;
#pragma unroll
          for (int jj = kk + 1; jj < 8; jj++)
            if (j0 + jj < ncols) v[jj] = __fma_rn(-l, T[(int64_t)k * ldt + j0 + jj], v[jj]);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; q++) row[q] = v[q];
    }
    __syncwarp();
  }
  // write back this warp's rows (pivot rows take their L11 row when pivpos is given)
  for (int r = 0; r < 16; r++) {
    int64_t gr = rbase + w * 16 + r;
    if (gr >= rows) break;
    int pp = pivpos ? pivpos[gr] : -1;
    const double* srow = pp >= 0 ? (L11 + (int64_t)pp * ldl11) : (Sw + r * lds);
    for (int c = lane; c < ncols; c += 32) out[gr * ldo + c] = srow[c];
  }
}

cudaError_t launch_trsm_rows(const double* A, int64_t lda, int64_t rows, int ncols, int nsub, const double* T,
                             int64_t ldt, const double* rdiag, double* out, int64_t ldo, const int* pivpos,
                             const double* L11, int64_t ldl11, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int ncp = (ncols + 7) & ~7;
  // rows per CTA: keep the tile <= ~100 KB (2 CTAs / SM)
  int nwarp = 4;
  while (nwarp > 1 && (size_t)16 * nwarp * (ncp + 4) * 8 > 100 * 1024) nwarp >>= 1;
  size_t smem = (size_t)16 * nwarp * (ncp + 4) * 8;
  int grid = (int)ceil_div<int64_t>(rows, 16 * nwarp);
  cudaError_t e;
  switch (nwarp) {
    case 4:
      e = cudaFuncSetAttribute(trsm_rows_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      trsm_rows_kernel<4><<<grid, 128, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
      break;
    case 2:
      e = cudaFuncSetAttribute(trsm_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      trsm_rows_kernel<2><<<grid, 64, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
      break;
    default:
      e = cudaFuncSetAttribute(trsm_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      trsm_rows_kernel<1><<<grid, 32, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ A * Tinv
// out = A Tinv with Tinv upper (zero lower part stored): the CholeskyQR2 tail
// V = W D^{-1}, Q = V J^{-1} (kappa(D) = kappa(W) <= ~7).  The CTA's rows
// are staged in shared memory first, so out may alias A.
template <int NWARP>
__global__ void __launch_bounds__(32 * NWARP)
rows_upper_kernel(const double* A, int64_t lda, int64_t rows, int n, const double* __restrict__ Tinv, double* out,
                  int64_t ldo) {
  extern __shared__ double S[];
  constexpr int TR = 16 * NWARP;
  const int ncp = (n + 7) & ~7;
  const int lds = ncp + 4;
  const int64_t rbase = (int64_t)blockIdx.x * TR;
  for (int idx = threadIdx.x; idx < TR * ncp; idx += blockDim.x) {
    int r = idx / ncp, c = idx - r * ncp;
    int64_t gr = rbase + r;
    S[r * lds + c] = (gr < rows && c < n) ? A[gr * lda + c] : 0.0;
  }
  __syncthreads();
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const double* Sw = S + (w * 16) * lds;
  for (int j0 = 0; j0 < ncp; j0 += 8) {
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int kend = min(j0 + 8, n);
    const bool colok = (j0 + g) < n;
    for (int k0 = 0; k0 < kend; k0 += 4) {
      const int k = k0 + t;
      double b = (k < kend && colok) ? Tinv[(int64_t)k * n + j0 + g] : 0.0;
#pragma unroll
      for (int mf = 0; mf < 2; mf++) {
        double a = Sw[(mf * 8 + g) * lds + k];
        dmma(acc[mf][0], acc[mf][1], a, b);
      }
    }
#pragma unroll
    for (int mf = 0; mf < 2; mf++) {
      int64_t gr = rbase + w * 16 + mf * 8 + g;
      int c = j0 + 2 * t;
      if (gr < rows) {
        if (c < n) out[gr * ldo + c] = acc[mf][0];
        if (c + 1 < n) out[gr * ldo + c + 1] = acc[mf][1];
      }
    }
  }
}

cudaError_t launch_rows_upper(const double* A, int64_t lda, int64_t rows, int n, const double* Tinv, double* out,
                              int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int ncp = (n + 7) & ~7;
  int nwarp = 4;
  while (nwarp > 1 && (size_t)16 * nwarp * (ncp + 4) * 8 > 100 * 1024) nwarp >>= 1;
  size_t smem = (size_t)16 * nwarp * (ncp + 4) * 8;
  int grid = (int)ceil_div<int64_t>(rows, 16 * nwarp);
  cudaError_t e;
  switch (nwarp) {
    case 4:
      e = cudaFuncSetAttribute(rows_upper_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      rows_upper_kernel<4><<<grid, 128, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
      break;
    case 2:
      e = cudaFuncSetAttribute(rows_upper_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      rows_upper_kernel<2><<<grid, 64, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
      break;
    default:
      e = cudaFuncSetAttribute(rows_upper_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      rows_upper_kernel<1><<<grid, 32, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Gram
// G = A^T A: 64 x 64 tiles of the upper triangle x split over rows.  Each CTA
// (4 warps, 32 x 32 each) streams 32-row chunks of the two column panels through
// shared memory and accumulates with DMMA; partial tiles go to `part` and a
// fixed-order reduction sums the splits and mirrors (exactly symmetric output).
constexpr int GT = 64, GK = 32;

struct GramGeom {
  int nt, ntiles, nsplit;
  int64_t rows_per_split;
};
static GramGeom gram_geom(int64_t rows, int n) {
  GramGeom g;
  g.nt = ceil_div(n, GT);
  g.ntiles = g.nt * (g.nt + 1) / 2;
  int64_t want = std::max<int64_t>(1, (2 * kSMs + g.ntiles - 1) / g.ntiles);
  int64_t maxs = std::max<int64_t>(1, rows / 256);
  g.nsplit = (int)std::min<int64_t>(want, maxs);
  g.rows_per_split = ceil_div<int64_t>(ceil_div<int64_t>(rows, g.nsplit), GK) * GK;
  g.nsplit = (int)std::max<int64_t>(1, ceil_div<int64_t>(rows, g.rows_per_split));
  return g;
}
size_t gram_partials_bytes(int64_t rows, int n) {
  GramGeom g = gram_geom(rows, n);
  return (size_t)g.nsplit * g.ntiles * GT * GT * sizeof(double);
}

__global__ void __launch_bounds__(128)
gram_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int n, int nt, int64_t rows_per_split,
            double* __restrict__ part) {
  __shared__ double Ai[GK][GT + 4];
  __shared__ double Aj[GK][GT + 4];
  // tile index -> (ti, tj), ti <= tj
  int tile = blockIdx.x, ti = 0;
  {
    int rem = tile;
    while (rem >= nt - ti) { rem -= nt - ti; ti++; }
    tile = rem + ti;  // tj
  }
  const int tj = tile;
  const int i0 = ti * GT, j0 = tj * GT;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = std::min<int64_t>(rows, r0 + rows_per_split);
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wi = (w >> 1) * 32, wj = (w & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t k0 = r0; k0 < r1; k0 += GK) {
    for (int idx = threadIdx.x; idx < GK * GT; idx += blockDim.x) {
      int kk = idx / GT, c = idx - kk * GT;
      int64_t gr = k0 + kk;
      bool rok = gr < r1;
      Ai[kk][c] = (rok && i0 + c < n) ? A[gr * lda + i0 + c] : 0.0;
      Aj[kk][c] = (rok && j0 + c < n) ? A[gr * lda + j0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = Ai[kk + t][wi + a * 8 + g];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = Aj[kk + t][wj + b * 8 + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
  double* P = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * GT * GT;
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) {
      int r = wi + a * 8 + g, c = wj + b * 8 + 2 * t;
      P[r * GT + c] = acc[a][b][0];
      P[r * GT + c + 1] = acc[a][b][1];
    }
}

// G[i][j] (i <= j) = sum over splits in fixed order, mirrored
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nsplit, int ntiles, int nt, int n,
                                   double* __restrict__ G) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (i > j) continue;
    int ti = i / GT, tj = j / GT;
    int tile = ti * nt - ti * (ti - 1) / 2 + (tj - ti);
    int r = i - ti * GT, c = j - tj * GT;
    double s = 0.0;
    for (int p = 0; p < nsplit; p++) s += part[((size_t)p * ntiles + tile) * GT * GT + r * GT + c];
    G[(int64_t)i * n + j] = s;
    G[(int64_t)j * n + i] = s;
  }
}

cudaError_t launch_gram(const double* A, int64_t lda, int64_t rows, int n, double* part, double* G, cudaStream_t st) {
  GramGeom gg = gram_geom(rows, n);
  dim3 grid(gg.ntiles, gg.nsplit);
  gram_kernel<<<grid, 128, 0, st>>>(A, lda, rows, n, gg.nt, gg.rows_per_split, part);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  int64_t total = (int64_t)n * n;
  gram_reduce_kernel<<<(int)std::min<int64_t>(ceil_div<int64_t>(total, 256), 1024), 256, 0, st>>>(part, gg.nsplit, gg.ntiles, gg.nt, n, G);
  return cudaGetLastError();
}

}  // namespace rlhc
