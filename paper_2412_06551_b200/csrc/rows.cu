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
  // rows are processed 4 at a time per thread with all loads issued before the tests
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < rows * n; base += 4 * stride) {
    double v[4];
    int64_t ee[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      ee[u] = base + u * stride;
      const int64_t i = ee[u] / n;
      v[u] = ee[u] < rows * n ? X[i * ldx + (ee[u] - i * n)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (!isfinite(v[u])) report(status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, ee[u]);
  }
}

cudaError_t launch_check_finite(const double* X, int64_t rows, int n, int64_t ldx, unsigned long long* status,
                                cudaStream_t st) {
  int64_t total = rows * n;
  int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), kSMs * 8);
  if (grid < 1) grid = 1;
  note_launch(); check_finite_kernel<<<grid, 256, 0, st>>>(X, rows, n, ldx, status);
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
  note_launch(); rdiag_kernel<<<ceil_div(n, 256), 256, 0, st>>>(T, n, ldt, rdiag, stage, status);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ substitution
// One warp owns 16 rows (two m8 fragments) of the CTA's row tile S (shared memory).
// Column block j0 (8 columns), with T[0:j0+8, j0:j0+8] and rdiag staged in shared
// memory (Tb, row stride 20 doubles: conflict-free B fragments):
//   acc = S[:, j0:j0+8]; acc += (-L[:, k]) T[k, j0:j0+8] for k < min(j0, nsub) (DMMA chain
//   in increasing k); then inside the 8-wide diagonal block the rows are substituted
//   in registers: l_k = acc_k * rdiag_k (broadcast by shuffle from the owning lane),
//   acc_j = fma(-l_k, T[k][j], acc_j) for j > k.  The fma chain per element is the
//   oracle's (DESIGN.md R#O5), so L is reproduced bit for bit.
constexpr int TB_LD = 20;

template <int NWARP>
__global__ void __launch_bounds__(32 * NWARP)
trsm_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int ncols, int nsub,
                 const double* __restrict__ T, int64_t ldt, const double* __restrict__ rdiag, double* out,
                 int64_t ldo, const int* __restrict__ pivpos, const double* __restrict__ L11, int64_t ldl11) {
  extern __shared__ double smem[];
  constexpr int TR = 16 * NWARP;
  const int ncp = (ncols + 7) & ~7;
  const int lds = ncp + 4;
  double* S = smem;                                   // TR x lds
  double* Tb = smem + TR * lds;                       // 2 x (ncp x TB_LD)
  double* rdb = Tb + 2 * ncp * TB_LD;                 // 2 x 8
  const int64_t rbase = (int64_t)blockIdx.x * TR;
  for (int idx = threadIdx.x; idx < TR * ncp; idx += blockDim.x) {
    int r = idx / ncp, c = idx - r * ncp;
    int64_t gr = rbase + r;
    S[r * lds + c] = (gr < rows && c < ncols) ? A[gr * lda + c] : 0.0;
  }
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  double* Sw = S + (w * 16) * lds;
  int buf = 0;
  for (int j0 = 0; j0 < ncp; j0 += 8, buf ^= 1) {
    // stage T[0 : min(j0+8, nsub), j0 : j0+8] and rdiag[j0 : j0+8]
    const int krows = min(j0 + 8, nsub);
    double* Tc = Tb + buf * ncp * TB_LD;
    for (int idx = threadIdx.x; idx < krows * 8; idx += blockDim.x) {
      int k = idx >> 3, c = idx & 7;
      Tc[k * TB_LD + c] = (j0 + c < ncols) ? T[(int64_t)k * ldt + j0 + c] : 0.0;
    }
    if (threadIdx.x < 8) rdb[buf * 8 + threadIdx.x] = (j0 + threadIdx.x < nsub) ? rdiag[j0 + threadIdx.x] : 0.0;
    __syncthreads();
    double acc[2][2];
#pragma unroll
    for (int mf = 0; mf < 2; mf++) {
      acc[mf][0] = Sw[(mf * 8 + g) * lds + j0 + 2 * t];
      acc[mf][1] = Sw[(mf * 8 + g) * lds + j0 + 2 * t + 1];
    }
    const int kend = min(j0, nsub);
#pragma unroll 2
    for (int k0 = 0; k0 < kend; k0 += 4) {
      const int k = k0 + t;
      const bool kok = k < kend;
      double b = kok ? Tc[k * TB_LD + g] : 0.0;
#pragma unroll
      for (int mf = 0; mf < 2; mf++) {
        double a = kok ? -Sw[(mf * 8 + g) * lds + k] : 0.0;
        dmma(acc[mf][0], acc[mf][1], a, b);
      }
    }
    if (j0 < nsub) {
      const double* Td = Tc + j0 * TB_LD;  // diagonal 8x8 block
#pragma unroll
      for (int kk = 0; kk < 8; kk++) {
        if (j0 + kk < nsub) {
          const double rk = rdb[buf * 8 + kk];
          const int src = (g << 2) | (kk >> 1);
          const double u0 = Td[kk * TB_LD + 2 * t], u1 = Td[kk * TB_LD + 2 * t + 1];
#pragma unroll
          for (int mf = 0; mf < 2; mf++) {
            double vk = __shfl_sync(0xffffffffu, (kk & 1) ? acc[mf][1] : acc[mf][0], src);
            double l = __dmul_rn(vk, rk);
            if (2 * t == kk) acc[mf][0] = l;
            else if (2 * t > kk) acc[mf][0] = __fma_rn(-l, u0, acc[mf][0]);
            if (2 * t + 1 == kk) acc[mf][1] = l;
            else if (2 * t + 1 > kk) acc[mf][1] = __fma_rn(-l, u1, acc[mf][1]);
          }
        }
      }
    }
#pragma unroll
    for (int mf = 0; mf < 2; mf++) {
      Sw[(mf * 8 + g) * lds + j0 + 2 * t] = acc[mf][0];
      Sw[(mf * 8 + g) * lds + j0 + 2 * t + 1] = acc[mf][1];
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

static size_t trsm_smem(int nwarp, int ncols) {
  const int ncp = (ncols + 7) & ~7;
  return ((size_t)16 * nwarp * (ncp + 4) + 2 * (size_t)ncp * TB_LD + 16) * sizeof(double);
}

cudaError_t launch_trsm_rows(const double* A, int64_t lda, int64_t rows, int ncols, int nsub, const double* T,
                             int64_t ldt, const double* rdiag, double* out, int64_t ldo, const int* pivpos,
                             const double* L11, int64_t ldl11, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  // without a pivot-row override the blocked path (same fma chain, much faster) is used
  if (!pivpos) return launch_trsm_blocked(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, st);
  const int ncp = (ncols + 7) & ~7;
  // rows per CTA: keep the tile <= ~100 KB (2 CTAs / SM)
  int nwarp = 4;
  while (nwarp > 1 && trsm_smem(nwarp, ncols) > 100 * 1024) nwarp >>= 1;
  size_t smem = trsm_smem(nwarp, ncols);
  (void)ncp;
  int grid = (int)ceil_div<int64_t>(rows, 16 * nwarp);
  cudaError_t e;
  switch (nwarp) {
    case 4:
      e = cudaFuncSetAttribute(trsm_rows_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      note_launch(); trsm_rows_kernel<4><<<grid, 128, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
      break;
    case 2:
      e = cudaFuncSetAttribute(trsm_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      note_launch(); trsm_rows_kernel<2><<<grid, 64, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
      break;
    default:
      e = cudaFuncSetAttribute(trsm_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      note_launch(); trsm_rows_kernel<1><<<grid, 32, smem, st>>>(A, lda, rows, ncols, nsub, T, ldt, rdiag, out, ldo, pivpos, L11, ldl11);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fused solve + Gram
// Persistent row-streaming kernel for n <= 128: out = A T^{-1} (substitution, the same
// per-element fma chain as trsm_rows_kernel, so L is still bit-exact) with
//   * T (n x n) and 1/diag(T) staged in shared memory once per CTA,
//   * row tiles of TR = 16*NWARP rows double-buffered with cp.async (the next tile
//     streams in while the current one is solved),
//   * optionally the Gram of the output accumulated on DMMA in registers
//     (CholeskyQR's G = W^T W fused into the pass that writes W: the pass reads its
//     input once and writes its output once), written as one n x n partial per CTA.
// out may equal A (each tile is read completely before it is written back).
constexpr int RS_MAXN = 128;
constexpr int RS_WARPS = 8;          // warps per CTA (2 CTAs per SM)
constexpr int RS_MF = 2;             // m8 fragments (16 rows) per warp
constexpr int RS_TR = 8 * RS_MF * RS_WARPS;  // rows per tile

// Asynchronous row-tile load: rows [row_base, row_base + nrows) x columns [0, ncp) of A
// into S (row stride lds), zero padded beyond `rows` / `ncols`.  Every thread issues all
// its 16-byte cp.async copies back to back (many loads in flight), then the caller waits.
__device__ __forceinline__ void tile_load_async(double* S, int lds, const double* A, int64_t lda, int64_t row_base,
                                                int64_t rows, int nrows, int ncols, int ncp, bool aligned) {
  const int nc2 = ncp >> 1;
  const int c2 = threadIdx.x % nc2, r0 = threadIdx.x / nc2, rstep = blockDim.x / nc2;
  if (r0 >= rstep) return;
  const int c = 2 * c2;
  const bool full = aligned && c + 1 < ncols;
  for (int r = r0; r < nrows; r += rstep) {
    const int64_t gr = row_base + r;
    double* dst = S + r * lds + c;
    const double* src = A + gr * lda + c;
    if (gr < rows && full) {
      cp_async16(dst, src);
    } else {
      dst[0] = (gr < rows && c < ncols) ? src[0] : 0.0;
      dst[1] = (gr < rows && c + 1 < ncols) ? src[1] : 0.0;
    }
  }
}

#ifdef RLHC_RS_TRACE
// probe builds only (tools/probe/prs.cu): per-phase timestamps of CTA 0, warp 0
__device__ long long g_rs_trace[256];
#define RS_TRACE(i)                                                                   \
  {                                                                                   \
    const int rs_i_ = (i);                                                            \
    if (blockIdx.x == 0 && threadIdx.x == 0 && rs_i_ < 256) g_rs_trace[rs_i_] = clock64(); \
  }
#else
#define RS_TRACE(i)
#endif

template <bool GRAM>
__global__ void __launch_bounds__(32 * RS_WARPS, 2)
rowsolve_kernel(const double* A, int64_t lda, int64_t rows, int n, const double* __restrict__ T, int64_t ldt,
                const double* __restrict__ rdiag, double* out, int64_t ldo, double* __restrict__ gpart) {
  // 8 warps x 16 rows: the substitution is a chain of dependent DMMA / fma steps per warp,
  // so throughput comes from the number of warps in flight (16 per SM)
  extern __shared__ double smem[];
  const int ncp = (n + 7) & ~7;
  const int lds = ncp + 4;        // == 4 (mod 16) doubles: conflict-free fragment access
  double* Tn = smem;              // -T, ncp x lds
  double* rd = Tn + ncp * lds;    // 1 / diag(T)
  double* S = rd + ncp;           // RS_TR x lds row tile
  // stage T with async copies (all in flight), then negate in shared memory
  tile_load_async(Tn, lds, T, ldt, 0, n, ncp, n, ncp, ((ldt & 1) == 0) && ((((uintptr_t)T) & 15) == 0));
  cp_async_commit();
  for (int k = threadIdx.x; k < ncp; k += blockDim.x) rd[k] = k < n ? rdiag[k] : 0.0;
  cp_async_wait_all();
  __syncthreads();
  for (int idx = threadIdx.x; idx < ncp * lds; idx += blockDim.x) Tn[idx] = -Tn[idx];
  const int64_t ntiles = ceil_div<int64_t>(rows, RS_TR);
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  // fused Gram (n <= 64): 32 x 32 output tiles of the upper triangle; tile (ti, tj) =
  // warp w & 3 (index 2, the lower tile, is unused), rows split in halves by w >> 2
  const int gt = (ncp + 31) / 32;
  const int gq = w & 3, ghalf = w >> 2;
  const int gti = gq >> 1, gtj = gq & 1;
  const bool gwork = GRAM && gti < gt && gtj < gt && gti <= gtj;
  double gacc[4][4][2];
  if (GRAM) {
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) gacc[a][b][0] = gacc[a][b][1] = 0.0;
  }
  const int nc2 = ncp >> 1;  // 16-byte chunks per row
  const bool aligned = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  double* Sw = S + (w * 8 * RS_MF) * lds;
  int trc = 1;
  RS_TRACE(0)
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t rbase = tile * RS_TR;
    __syncthreads();  // previous tile fully consumed
    // ---- load the row tile (async 16-byte copies, zero padding)
    tile_load_async(S, lds, A, lda, rbase, rows, RS_TR, n, ncp, aligned);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    RS_TRACE(trc++)
    // ---- substitution, column blocks of 8
    for (int j0 = 0; j0 < ncp; j0 += 8) {
      double acc[RS_MF][2];
#pragma unroll
      for (int mf = 0; mf < RS_MF; mf++) {
        const double2 c2 = *reinterpret_cast<const double2*>(Sw + (mf * 8 + g) * lds + j0 + 2 * t);
        acc[mf][0] = c2.x; acc[mf][1] = c2.y;
      }
#pragma unroll 2
      for (int k0 = 0; k0 < j0; k0 += 4) {
        const double b = Tn[(k0 + t) * lds + j0 + g];
#pragma unroll
        for (int mf = 0; mf < RS_MF; mf++) dmma(acc[mf][0], acc[mf][1], Sw[(mf * 8 + g) * lds + k0 + t], b);
      }
#pragma unroll
      for (int mf = 0; mf < RS_MF; mf++)
        *reinterpret_cast<double2*>(Sw + (mf * 8 + g) * lds + j0 + 2 * t) = make_double2(acc[mf][0], acc[mf][1]);
      __syncwarp();
      // diagonal 8x8 block: lane = row (16 rows per warp), static indices:
      //   l_k = v_k * (1/T_kk);  v_j = fma(l_k, -T_kj, v_j)  (== fma(-l_k, T_kj, v_j))
      if (lane < 8 * RS_MF) {
        double* row = Sw + lane * lds + j0;
        double v[8];
        {
          const double2 p0 = reinterpret_cast<const double2*>(row)[0], p1 = reinterpret_cast<const double2*>(row)[1];
          const double2 p2 = reinterpret_cast<const double2*>(row)[2], p3 = reinterpret_cast<const double2*>(row)[3];
          v[0] = p0.x; v[1] = p0.y; v[2] = p1.x; v[3] = p1.y; v[4] = p2.x; v[5] = p2.y; v[6] = p3.x; v[7] = p3.y;
        }
        const double* Td = Tn + j0 * lds + j0;
        const int kmax = min(8, n - j0);
#pragma unroll
        for (int kk = 0; kk < 8; kk++) {
          if (kk < kmax) {
            const double l = __dmul_rn(v[kk], rd[j0 + kk]);
            v[kk] = l;
#pragma unroll
            for (int jj = kk + 1; jj < 8; jj++) v[jj] = __fma_rn(l, Td[kk * lds + jj], v[jj]);
          }
        }
        reinterpret_cast<double2*>(row)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(row)[1] = make_double2(v[2], v[3]);
        reinterpret_cast<double2*>(row)[2] = make_double2(v[4], v[5]);
        reinterpret_cast<double2*>(row)[3] = make_double2(v[6], v[7]);
      }
      __syncwarp();
    }
    RS_TRACE(trc++)
    __syncthreads();
    // ---- store the tile (16-byte stores; out == nullptr: the Gram only)
    if (out) {
      const int c2 = threadIdx.x % nc2, r0 = threadIdx.x / nc2, rstep = blockDim.x / nc2;
      const int c = 2 * c2;
      const bool ofull = c + 1 < n && ((ldo & 1) == 0) && ((((uintptr_t)out) & 15) == 0);
      if (r0 < rstep)
        for (int r = r0; r < RS_TR; r += rstep) {
          const int64_t gr = rbase + r;
          if (gr >= rows) break;
          const double2 v = *reinterpret_cast<const double2*>(S + r * lds + c);
          double* dst = out + gr * ldo + c;
          if (ofull) *reinterpret_cast<double2*>(dst) = v;
          else { if (c < n) dst[0] = v.x; if (c + 1 < n) dst[1] = v.y; }
        }
    }
    RS_TRACE(trc++)
    if (gwork) {
      // G += tile^T tile on DMMA (rows beyond `rows` are zero-padded); this warp: rows
      // [ghalf * RS_TR/2, (ghalf+1) * RS_TR/2) of its 32 x 32 tile
      const int i0 = gti * 32, j0 = gtj * 32;
      const int kb = ghalf * (RS_TR / 2);
#pragma unroll 2
      for (int k0 = kb; k0 < kb + RS_TR / 2; k0 += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int a = 0; a < 4; a++) af[a] = (i0 + a * 8 < ncp) ? S[(k0 + t) * lds + i0 + a * 8 + g] : 0.0;
#pragma unroll
        for (int b = 0; b < 4; b++) bf[b] = (j0 + b * 8 < ncp) ? S[(k0 + t) * lds + j0 + b * 8 + g] : 0.0;
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) dmma(gacc[a][b][0], gacc[a][b][1], af[a], bf[b]);
      }
    }
  }
  RS_TRACE(trc++)
  if (GRAM) {
    // the two row halves of each tile: half 1 -> shared memory, half 0 adds it (fixed order)
    __syncthreads();
    double* Gs = S;  // reuse the tile buffer: 4 tiles x 32 x 33
    if (gwork && ghalf == 1) {
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
          const int r = a * 8 + g, c = b * 8 + 2 * t;
          Gs[gq * 32 * 33 + r * 33 + c] = gacc[a][b][0];
          Gs[gq * 32 * 33 + r * 33 + c + 1] = gacc[a][b][1];
        }
    }
    __syncthreads();
    if (gwork && ghalf == 0) {
      double* P = gpart + (size_t)blockIdx.x * ncp * ncp;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
          const int r = a * 8 + g, c = b * 8 + 2 * t;
          const int gr = gti * 32 + r, gc = gtj * 32 + c;
          if (gr < ncp && gc < ncp) {
            P[gr * ncp + gc] = gacc[a][b][0] + Gs[gq * 32 * 33 + r * 33 + c];
            P[gr * ncp + gc + 1] = gacc[a][b][1] + Gs[gq * 32 * 33 + r * 33 + c + 1];
          }
        }
    }
  }
}

// pivot rows of L take their L11 row (exact unit diagonal, DESIGN.md R#O5)
__global__ void pivot_rows_kernel(const int64_t* __restrict__ piv, int n, int64_t row0, int64_t rows,
                                  const double* __restrict__ L11, double* out, int64_t ldo) {
  const int k = blockIdx.x;
  const int64_t lr = piv[k] - row0;
  if (lr < 0 || lr >= rows) return;
  for (int c = threadIdx.x; c < n; c += blockDim.x) out[lr * ldo + c] = L11[(int64_t)k * n + c];
}

// G[i][j] = sum over CTA partials in fixed order (8 independent partial sums, then a
// fixed combination), upper triangle, mirrored -> exactly symmetric
__global__ void __launch_bounds__(256)
gram_part_reduce_kernel(const double* __restrict__ part, int nparts, int n, int ncp, double* __restrict__ G) {
  // block = 32 consecutive elements of the ncp x ncp partial layout x 8 warps; warp q sums
  // partials [q*per, (q+1)*per) with 8 independent accumulators (loads in flight), then the
  // 8 warp sums are combined in a fixed order: deterministic for a given launch geometry.
  __shared__ double red[8][32];
  const int lane = lane_id(), wq = warp_id();
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int64_t total = (int64_t)ncp * ncp;
  const int per = (nparts + 7) / 8;
  const int p0 = wq * per, p1 = min(nparts, p0 + per);
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (e < total) {
    const double* p = part + e;
    int q = p0;
    for (; q + 8 <= p1; q += 8)
#pragma unroll
      for (int u = 0; u < 8; u++) s[u] += p[(size_t)(q + u) * total];
    for (; q < p1; q++) s[0] += p[(size_t)q * total];
  }
  red[wq][lane] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  __syncthreads();
  if (wq == 0 && e < total) {
    double v = red[0][lane];
    for (int q = 1; q < 8; q++) v += red[q][lane];
    const int i = (int)(e / ncp), j = (int)(e - (int64_t)i * ncp);
    if (i < n && j < n && i <= j) {
      G[(int64_t)i * n + j] = v;
      G[(int64_t)j * n + i] = v;
    }
  }
}

cudaError_t launch_pivot_rows(const int64_t* piv, int n, int64_t row0, int64_t rows, const double* L11, double* out,
                              int64_t ldo, cudaStream_t st) {
  note_launch();
  pivot_rows_kernel<<<n, 64, 0, st>>>(piv, n, row0, rows, L11, out, ldo);
  return cudaGetLastError();
}

static size_t rowsolve_smem(int n) {
  const int ncp = (n + 7) & ~7, lds = ncp + 4;
  return ((size_t)ncp * lds + ncp + (size_t)RS_TR * lds) * sizeof(double);
}
static int rowsolve_grid(int64_t rows, int n) {
  const int64_t ntiles = ceil_div<int64_t>(rows, RS_TR);
  const int per_sm = rowsolve_smem(n) > 110 * 1024 ? 1 : 2;
  return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)kSMs * per_sm));
}
bool rowsolve_ok(int n) { return n <= 64; }
size_t rowsolve_partials_bytes(int64_t rows, int n) {
  const int ncp = (n + 7) & ~7;
  return (size_t)rowsolve_grid(rows, n) * ncp * ncp * sizeof(double);
}

template <bool GRAM>
static cudaError_t run_rowsolve(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                                const double* rdiag, double* out, int64_t ldo, double* gpart, cudaStream_t st) {
  size_t smem = rowsolve_smem(n);
  cudaError_t e = cudaFuncSetAttribute(rowsolve_kernel<GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  note_launch();
  rowsolve_kernel<GRAM><<<rowsolve_grid(rows, n), 32 * RS_WARPS, smem, st>>>(A, lda, rows, n, T, ldt, rdiag, out,
                                                                            ldo, gpart);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ blocked TRSM (n > 64)
// C_out = C_in - A B (rows x N, K <= 64) on DMMA, the chain over k in increasing order:
// Cout = Cin - A B (rows x N, A rows x K, B K x N) on DMMA: the updates of the blocked
// substitution and factorizations.  Every element is Cin followed by the fma chain over
// k = 0, 1, ..., K-1 in increasing order (DMMA m8n8k4 == the fma chain k0..k3; zero-padded k
// leaves the value unchanged), i.e. the substitution's own chain.  CTA tile 128 x 64, 8 warps
// of 32 x 32, K chunks of 32 double-buffered with cp.async, 2 CTAs per SM.
constexpr int GS_M = 128, GS_N = 64, GS_K = 32;
struct GemmSmem {
  double A[2][GS_M][GS_K + 4];
  double B[2][GS_K][GS_N + 4];
};

__global__ void __launch_bounds__(256, 2)
gemm_sub_kernel(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* __restrict__ A,
                int64_t lda, const double* __restrict__ B, int64_t ldb, int64_t rows, int K, int N) {
  extern __shared__ __align__(16) unsigned char gs_raw[];
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>(gs_raw);
  const int64_t r0 = (int64_t)blockIdx.x * GS_M;
  const int c0 = blockIdx.y * GS_N;
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wi = (w >> 1) * 32, wj = (w & 1) * 32;
  const bool al_a = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  const bool al_b = ((ldb & 1) == 0) && ((((uintptr_t)B) & 15) == 0);
  const bool full_rows = r0 + GS_M <= rows, full_cols = c0 + GS_N <= N;
  auto load_chunk = [&](int st, int kc) {
    const bool full_k = kc + GS_K <= K;
    // A: 128 rows x 32 k = 2048 pairs, 8 per thread
#pragma unroll
    for (int i = 0; i < GS_M * GS_K / 2 / 256; i++) {
      const int idx = threadIdx.x + 256 * i;
      const int r = idx / (GS_K / 2), c = 2 * (idx % (GS_K / 2));
      const int64_t gr = r0 + r;
      const int k = kc + c;
      double* dst = &sm.A[st][r][c];
      const double* src = A + gr * lda + k;
      if (al_a && full_rows && full_k) {
        cp_async16(dst, src);
      } else {
        const bool rok = gr < rows;
        cp_async8(dst, (rok && k < K) ? src : A, (rok && k < K) ? 8 : 0);
        cp_async8(dst + 1, (rok && k + 1 < K) ? src + 1 : A, (rok && k + 1 < K) ? 8 : 0);
      }
    }
    // B: 32 k x 64 columns = 1024 pairs, 4 per thread
#pragma unroll
    for (int i = 0; i < GS_K * GS_N / 2 / 256; i++) {
      const int idx = threadIdx.x + 256 * i;
      const int r = idx / (GS_N / 2), c = 2 * (idx % (GS_N / 2));
      const int k = kc + r;
      double* dst = &sm.B[st][r][c];
      const double* src = B + (int64_t)k * ldb + c0 + c;
      if (al_b && full_cols && full_k) {
        cp_async16(dst, src);
      } else {
        const bool kok = k < K;
        cp_async8(dst, (kok && c0 + c < N) ? src : B, (kok && c0 + c < N) ? 8 : 0);
        cp_async8(dst + 1, (kok && c0 + c + 1 < N) ? src + 1 : B, (kok && c0 + c + 1 < N) ? 8 : 0);
      }
    }
    cp_async_commit();
  };
  if (K > 0) load_chunk(0, 0);
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int64_t gr = r0 + wi + a * 8 + g;
      const int c = c0 + wj + b * 8 + 2 * t;
      acc[a][b][0] = (gr < rows && c < N) ? Cin[gr * ldci + c] : 0.0;
      acc[a][b][1] = (gr < rows && c + 1 < N) ? Cin[gr * ldci + c + 1] : 0.0;
    }
  int st = 0;
  for (int kc = 0; kc < K; kc += GS_K) {
    if (kc + GS_K < K) {
      load_chunk(st ^ 1, kc + GS_K);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll
    for (int k0 = 0; k0 < GS_K; k0 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = -sm.A[st][wi + a * 8 + g][k0 + t];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = sm.B[st][k0 + t][wj + b * 8 + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
    st ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int64_t gr = r0 + wi + a * 8 + g;
      const int c = c0 + wj + b * 8 + 2 * t;
      if (gr < rows) {
        if (c < N) Cout[gr * ldco + c] = acc[a][b][0];
        if (c + 1 < N) Cout[gr * ldco + c + 1] = acc[a][b][1];
      }
    }
}

cudaError_t launch_gemm_update(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                               int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N, cudaStream_t st) {
  if (rows <= 0 || N <= 0) return cudaSuccess;
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, gemm_sub_kernel, (int)sizeof(GemmSmem))) return e;
  dim3 grid((unsigned)ceil_div<int64_t>(rows, GS_M), (unsigned)ceil_div(N, GS_N));
  note_launch();
  gemm_sub_kernel<<<grid, 256, sizeof(GemmSmem), st>>>(Cin, ldci, Cout, ldco, A, lda, B, ldb, rows, K, N);
  return cudaGetLastError();
}

// out = A T^{-1} (rows x n, substitution, the oracle's fma chain) for any n: panels of 64
// columns solved by rowsolve_kernel, each followed by the DMMA update of the trailing columns.
// With nsub < n only the first nsub columns are substituted (the rest receive the updates):
// the elimination step of a tournament panel.
cudaError_t launch_trsm_blocked(const double* A, int64_t lda, int64_t rows, int n, int nsub, const double* T,
                                int64_t ldt, const double* rdiag, double* out, int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  // left-looking: panel p0 = A(:, p0:p0+w) - out(:, 0:p0) T(0:p0, p0:p0+w) (one GEMM, k in
  // increasing order -- the same chain as updating panel by panel), then its substitution
  for (int p0 = 0; p0 < nsub; p0 += 64) {
    const int w = std::min(64, nsub - p0);
    cudaError_t e;
    if (p0 > 0) {
      e = launch_gemm_update(A + p0, lda, out + p0, ldo, out, ldo, T + p0, ldt, rows, p0, w, st);
      if (e) return e;
    }
    const double* src = (p0 == 0) ? A : out;
    const int64_t lds_ = (p0 == 0) ? lda : ldo;
    e = run_rowsolve<false>(src + p0, lds_, rows, w, T + (int64_t)p0 * ldt + p0, ldt, rdiag + p0, out + p0, ldo,
                            nullptr, st);
    if (e) return e;
  }
  // columns past nsub receive the updates of every substituted column
  if (nsub < n) return launch_gemm_update(A + nsub, lda, out + nsub, ldo, out, ldo, T + nsub, ldt, rows, nsub, n - nsub, st);
  return cudaSuccess;
}

cudaError_t launch_rowsolve(const double* A, int64_t lda, int64_t rows, int n, const double* T, const double* rdiag,
                            double* out, int64_t ldo, const int64_t* piv, const double* L11, double* gpart, double* G,
                            cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const bool gram = G != nullptr;
  cudaError_t e = gram ? run_rowsolve<true>(A, lda, rows, n, T, n, rdiag, out, ldo, gpart, st)
                       : run_rowsolve<false>(A, lda, rows, n, T, n, rdiag, out, ldo, gpart, st);
  if (e) return e;
  if (piv) {
    note_launch();
    pivot_rows_kernel<<<n, 64, 0, st>>>(piv, n, 0, rows, L11, out, ldo);
  }
  if (!gram) return cudaGetLastError();
  const int ncp = (n + 7) & ~7;
  int64_t total = (int64_t)n * n;
  note_launch();
  (void)total;
  gram_part_reduce_kernel<<<(int)ceil_div<int64_t>((int64_t)ncp * ncp, 32), 256, 0, st>>>(gpart, rowsolve_grid(rows, n),
                                                                                          n, ncp, G);
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
      note_launch(); rows_upper_kernel<4><<<grid, 128, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
      break;
    case 2:
      e = cudaFuncSetAttribute(rows_upper_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      note_launch(); rows_upper_kernel<2><<<grid, 64, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
      break;
    default:
      e = cudaFuncSetAttribute(rows_upper_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      note_launch(); rows_upper_kernel<1><<<grid, 32, smem, st>>>(A, lda, rows, n, Tinv, out, ldo);
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
  // 3 resident CTAs per SM (68 KB of shared memory each), split count rounded so the last
  // wave is (nearly) full
  const int64_t slots = 3 * (int64_t)kSMs;
  int64_t want = std::max<int64_t>(1, (slots + g.ntiles - 1) / g.ntiles);
  want = std::max<int64_t>(1, ((want * g.ntiles + slots - 1) / slots) * slots / g.ntiles);
  int64_t maxs = std::max<int64_t>(1, rows / 256);
  g.nsplit = (int)std::min<int64_t>(want, maxs);
  g.rows_per_split = ceil_div<int64_t>(ceil_div<int64_t>(rows, g.nsplit), GK) * GK;
  g.nsplit = (int)std::max<int64_t>(1, ceil_div<int64_t>(rows, g.rows_per_split));
  return g;
}
size_t gram_partials_bytes(int64_t rows, int n) {
  GramGeom g = gram_geom(rows, n);
  return std::max((size_t)g.nsplit * g.ntiles * GT * GT * sizeof(double), syrk_partials_bytes(n));
}

__global__ void __launch_bounds__(128, 3)
gram_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int n, int nt, int64_t rows_per_split,
            double* __restrict__ part) {
  // two chunks in flight: the next chunk's column panels stream in (cp.async) while the
  // current one is contracted
  extern __shared__ __align__(16) double gram_sm[];
  double(*Ai)[GK][GT + 4] = reinterpret_cast<double(*)[GK][GT + 4]>(gram_sm);
  double(*Aj)[GK][GT + 4] = reinterpret_cast<double(*)[GK][GT + 4]>(gram_sm + 2 * GK * (GT + 4));
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
  // a diagonal tile's lower 32 x 32 quarter is never used (G is mirrored from its upper
  // triangle, gram_reduce_kernel): that warp skips its contraction
  const bool lower_warp = ti == tj && wi > wj;
  // ... and in a diagonal 32 x 32 quarter the fragments strictly below the diagonal (a > b)
  const bool diag_warp = ti == tj && wi == wj;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const bool aligned = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  // interior chunks (all GK rows in range, both 64-column panels inside n): thread
  // (warp w, lane) copies rows w + 4j, columns 2*lane, 2*lane+1 of each panel -- no
  // per-copy index arithmetic or bounds tests
  const bool cols_full = aligned && i0 + GT <= n && j0 + GT <= n;
  auto fetch = [&](int64_t k0, int buf) {
    if (cols_full && k0 + GK <= r1) {
      const double* pi = A + (k0 + w) * lda + i0 + 2 * lane;
      const double* pj = A + (k0 + w) * lda + j0 + 2 * lane;
      const int64_t step = 4 * lda;
#pragma unroll
      for (int j = 0; j < GK / 4; j++) {
        cp_async16(&Ai[buf][w + 4 * j][2 * lane], pi + j * step);
        cp_async16(&Aj[buf][w + 4 * j][2 * lane], pj + j * step);
      }
      cp_async_commit();
      return;
    }
    for (int idx = threadIdx.x; idx < GK * (GT / 2); idx += blockDim.x) {
      const int kk = idx / (GT / 2), c = 2 * (idx % (GT / 2));
      const int64_t gr = k0 + kk;
      const bool rok = gr < r1;
#pragma unroll
      for (int side = 0; side < 2; side++) {
        const int cb = side ? j0 : i0;
        double* dst = side ? &Aj[buf][kk][c] : &Ai[buf][kk][c];
        const double* src = A + gr * lda + cb + c;
        if (rok && aligned && cb + c + 1 < n) cp_async16(dst, src);
        else {
          dst[0] = (rok && cb + c < n) ? src[0] : 0.0;
          dst[1] = (rok && cb + c + 1 < n) ? src[1] : 0.0;
        }
      }
    }
    cp_async_commit();
  };
  if (r0 < r1) fetch(r0, 0);
  int buf = 0;
  for (int64_t k0 = r0; k0 < r1; k0 += GK, buf ^= 1) {
    if (k0 + GK < r1) {
      fetch(k0 + GK, buf ^ 1);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = Ai[buf][kk + t][wi + a * 8 + g];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = Aj[buf][kk + t][wj + b * 8 + g];
      if (diag_warp) {
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++)
            if (a <= b)
              asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                  : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                  : "d"(af[a]), "d"(bf[b]));
      } else if (!lower_warp) {
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                : "d"(af[a]), "d"(bf[b]));
      }
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
  bool done = false;  // n <= 256, TMA-describable A: the fragment-balanced TMA kernel (syrk.cu)
  if (cudaError_t e = launch_syrk(A, lda, rows, n, part, G, st, &done)) return e;
  if (done) return cudaSuccess;
  GramGeom gg = gram_geom(rows, n);
  dim3 grid(gg.ntiles, gg.nsplit);
  constexpr int smem = 4 * GK * (GT + 4) * (int)sizeof(double);
  static DevFlags attr;
  if (cudaError_t e0 = smem_attr(attr, gram_kernel, smem)) return e0;
  note_launch(); gram_kernel<<<grid, 128, smem, st>>>(A, lda, rows, n, gg.nt, gg.rows_per_split, part);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  int64_t total = (int64_t)n * n;
  note_launch(); gram_reduce_kernel<<<(int)std::min<int64_t>(ceil_div<int64_t>(total, 256), 1024), 256, 0, st>>>(part, gg.nsplit, gg.ntiles, gg.nt, n, G);
  return cudaGetLastError();
}

}  // namespace rlhc

namespace rlhc {

// ------------------------------------------------------------------ substitution, oracle op order
// out = A T^{-1} (T upper, n <= 64) with the oracle's operation sequence (ora_trsm_right_upper,
// DESIGN.md R#O9): acc = a_k; acc = acc - (o_j * T[j][k]) for j < k (a rounded product, then a
// rounded difference: no fma); o_k = acc / T[k][k] (IEEE division).  Used for W = X Y^{-1}
// (n > 64: subst.cu) -- the CholeskyQR passes V = W D^-1, Q = V J^-1 keep the fma
// chain (rowsolve_kernel) or, for n > 64, the explicit inverse (R#9): the fma chain amplifies
// cancellation in W on the arrowhead of P:1071-1082 (|W| 1.5e10 instead of 19 at beta =
// 1e-25, tools/arrow_fma.py), this sequence does not; W is bit-identical to the oracle's.  Thread per row, the
// row in registers (static indices), T in shared memory (broadcast reads), row tiles staged
// through shared memory with coalesced cp.async; out may alias A.
constexpr int SMS_R = 128, SMS_LD = 65;
__host__ __device__ inline int sms_smem_bytes() { return (64 * 64 + 128 + SMS_R * SMS_LD) * (int)sizeof(double); }
// a / b correctly rounded (== __ddiv_rn) from y = RN(1/b): q0 = RN(a y) is within 1.5 ulp of
// a/b, one residual step q1 = q0 + (a - b q0) y brings it within 1 ulp, and by Markstein's
// theorem (y within 1/2 ulp of 1/b, q1 within 1 ulp of a/b, r1 = a - b q1 exact) the second
// step RN(q1 + r1 y) is RN(a/b).  Five dependent FP64 ops instead of the library sequence;
// away from the exponent range where the theorem's no-underflow/overflow premise holds
// (and for a zero quotient, to keep the sign of zero) the library division is used.
RLHC_DEV double div_by_rcp(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q1 = __fma_rn(__fma_rn(-b, q0, a), y, q0);
  const double q2 = __fma_rn(__fma_rn(-b, q1, a), y, q1);
  const double aa = fabs(a), aq = fabs(q2);
  if (aa >= 0x1p-900 && aa <= 0x1p+900 && aq >= 0x1p-900 && aq <= 0x1p+900) return q2;
  return __ddiv_rn(a, b);
}
// Persistent: each CTA stages T^T once, then loops over 128-row tiles; with GRAM the CTA
// accumulates its partial W^T W of the upper 32 x 32 tiles on DMMA from the solved tile
// (warp q < 3: tile (0,0), (0,1), (1,1)), reduced by gram_part_reduce_kernel.
// Right-looking with ROTATED registers: at step k, acc[c] holds column k + c of the row, so
// acc[0] is divided by T_kk and every later column receives - o_k T[k][k+c] (a rounded
// product, then a rounded difference): per element the same terms in the same (increasing
// j) order as the oracle's left-looking loop.  A compact loop (the fully unrolled
// triangle was instruction-bound), up to 63 independent updates per step; the rotation
// narrows to 48, 32, 16 slots as the live columns shrink.
template <int NS>
RLHC_DEV void sms_steps(double (&acc)[64], int k0, int k1, const double* Tsh, const double* diag, double* orow) {
#pragma unroll 1
  for (int k = k0; k < k1; k++) {
    const double wk = div_by_rcp(acc[0], diag[k], diag[64 + k]);
    orow[k] = wk;
    const double* u = Tsh + k * 64;  // u[c] = T[k][k + 1 + c] (0 past n)
#pragma unroll
    for (int c = 0; c < NS - 1; c += 2) {
      const double2 uu = *reinterpret_cast<const double2*>(u + c);
      acc[c] = __dsub_rn(acc[c + 1], __dmul_rn(wk, uu.x));
      if (c + 1 < NS - 1) acc[c + 1] = __dsub_rn(acc[c + 2], __dmul_rn(wk, uu.y));
    }
    acc[NS - 1] = 0.0;
  }
}
template <bool GRAM>
__global__ void __launch_bounds__(SMS_R, 2)
subst_ms_kernel(const double* A, int64_t lda, int64_t rows, int n, const double* __restrict__ T, int64_t ldt,
                double* out, int64_t ldo, double* __restrict__ gpart) {
  extern __shared__ __align__(16) double sms[];
  double* Tsh = sms;              // [64][64]: Tsh[k][c] = T[k][k + 1 + c]
  double* diag = Tsh + 64 * 64;   // [128]: T_kk, then RN(1 / T_kk)
  double* tile = diag + 128;      // [SMS_R][SMS_LD]
  const int tid = threadIdx.x, lane = lane_id(), wq = warp_id();
  const int g = lane >> 2, t = lane & 3;
  for (int e = tid; e < 64 * 64; e += SMS_R) {  // all loads in flight (cp.async, zero fill)
    const int k = e >> 6, c = e & 63, j = k + 1 + c;
    const bool in = k < n && j < n;
    cp_async8(Tsh + e, in ? T + (int64_t)k * ldt + j : T, in ? 8 : 0);
  }
  cp_async_commit();
  if (tid < 64) {  // diag[k] = T_kk, diag[64 + k] = RN(1 / T_kk) (NaN outside div_by_rcp's range)
    const double d = tid < n ? T[(int64_t)tid * ldt + tid] : 1.0;
    const double ad = fabs(d);
    diag[tid] = d;
    diag[64 + tid] = (ad >= 0x1p-900 && ad <= 0x1p+900) ? __drcp_rn(d) : __longlong_as_double(0x7ff8000000000000LL);
  }
  const int ncp = (n + 7) & ~7;
  const int gt = (ncp + 31) / 32;
  const int gti = wq >> 1, gtj = (wq == 0) ? 0 : 1;  // warp 0: (0,0), 1: (0,1), 2: (1,1)
  const bool gwork = GRAM && wq < 3 && gtj < gt && gti < gt;
  double gacc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) gacc[a][b][0] = gacc[a][b][1] = 0.0;
  const int64_t ntiles = ceil_div<int64_t>(rows, SMS_R);
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t r0 = tl * SMS_R;
    __syncthreads();  // previous tile consumed (stores and Gram)
    for (int e = tid; e < SMS_R * 64; e += SMS_R) {
      const int q = e >> 6, c = e & 63;
      const bool in = r0 + q < rows && c < n;
      cp_async8(tile + q * SMS_LD + c, in ? A + (r0 + q) * lda + c : A, in ? 8 : 0);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    double acc[64];
    double* orow = tile + tid * SMS_LD;
#pragma unroll
    for (int c = 0; c < 64; c++) acc[c] = orow[c];
    // at step k the live columns are k .. n-1: rotate 64, 48, 32, 16 slots as they shrink
    sms_steps<64>(acc, 0, min(n, 16), Tsh, diag, orow);
    sms_steps<48>(acc, min(n, 16), min(n, 32), Tsh, diag, orow);
    sms_steps<32>(acc, min(n, 32), min(n, 48), Tsh, diag, orow);
    sms_steps<16>(acc, min(n, 48), n, Tsh, diag, orow);
    __syncthreads();
    for (int e = tid; e < SMS_R * 64; e += SMS_R) {
      const int q = e >> 6, c = e & 63;
      if (r0 + q < rows && c < n) out[(r0 + q) * ldo + c] = tile[q * SMS_LD + c];
    }
    if (gwork) {  // G(ti, tj) += W(:, ti block)^T W(:, tj block) over the tile's rows
#pragma unroll 2
      for (int k0 = 0; k0 < SMS_R; k0 += 4) {
        double af[4], bf[4];
        const double* rowp = tile + (k0 + t) * SMS_LD;
#pragma unroll
        for (int a = 0; a < 4; a++) af[a] = rowp[gti * 32 + a * 8 + g];
#pragma unroll
        for (int b = 0; b < 4; b++) bf[b] = rowp[gtj * 32 + b * 8 + g];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++) dmma(gacc[a][b][0], gacc[a][b][1], af[a], bf[b]);
      }
    }
  }
  if (gwork) {
    double* P = gpart + (size_t)blockIdx.x * ncp * ncp;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int gr = gti * 32 + a * 8 + g, gc = gtj * 32 + b * 8 + 2 * t;
        if (gr < ncp && gc < ncp) {
          P[gr * ncp + gc] = gacc[a][b][0];
          P[gr * ncp + gc + 1] = gacc[a][b][1];
        }
      }
  }
}

static int sms_grid(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, SMS_R), (int64_t)kSMs * 2));
}
size_t subst_ms_partials_bytes(int64_t rows, int n) {
  const int ncp = (n + 7) & ~7;
  return (size_t)sms_grid(rows) * ncp * ncp * sizeof(double);
}

bool subst_ms_ok(int n) { return n <= 64; }

cudaError_t launch_subst_ms(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                            double* out, int64_t ldo, double* gpart, double* G, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int smem = sms_smem_bytes();
  static DevFlags attr_t, attr_f;
  if (cudaError_t e = smem_attr(attr_t, subst_ms_kernel<true>, smem)) return e;
  if (cudaError_t e = smem_attr(attr_f, subst_ms_kernel<false>, smem)) return e;
  const int grid = sms_grid(rows);
  note_launch();
  if (G) subst_ms_kernel<true><<<grid, SMS_R, smem, st>>>(A, lda, rows, n, T, ldt, out, ldo, gpart);
  else subst_ms_kernel<false><<<grid, SMS_R, smem, st>>>(A, lda, rows, n, T, ldt, out, ldo, gpart);
  if (!G) return cudaGetLastError();
  const int ncp = (n + 7) & ~7;
  note_launch();
  gram_part_reduce_kernel<<<(int)ceil_div<int64_t>((int64_t)ncp * ncp, 32), 256, 0, st>>>(gpart, grid, n, ncp, G);
  return cudaGetLastError();
}

}  // namespace rlhc
