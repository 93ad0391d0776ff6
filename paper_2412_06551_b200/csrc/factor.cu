// factor.cu -- the small n x n / s x n factorizations (replicated work, no m dependence):
// HouseholderQR of the sketch (only R kept, H never formed) and Cholesky with
// breakdown detection.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

// ------------------------------------------------------------------ Householder R
// LAPACK dgeqr2 order (DESIGN.md R#O7): beta = -sign(alpha) ||x||, tau = (beta - alpha)/beta,
// v = x(2:)/(alpha - beta); A(k:, k+1:) -= tau v (v^T A(k:, k+1:)).
// One CTA, column j owned by warp (j mod NW).  Look-ahead: in step k every warp applies
// reflector k to its columns; the owner of column k+1 does that column first and then
// immediately forms reflector k+1 (norm, beta, tau, v scaled in place) and publishes
// (beta, tau) -- so one barrier per step and the reflector never waits for the other
// columns.  Working copy with row stride n+1 (conflict-free column access); explicit
// shared memory when it fits (SMEM), else global `work`.
template <bool SMEM>
__global__ void __launch_bounds__(1024)
hqr2_kernel(const double* __restrict__ A, int s, int n, int64_t lda, const double* __restrict__ sgn_ref,
            double* __restrict__ S, double* __restrict__ work, unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ double tauS[2];
  __shared__ int flag;
  double* Wm = SMEM ? dsm : work;
  const int ld = n + 1;
  const int lane = lane_id(), wp = warp_id(), nw = blockDim.x >> 5;
  for (int i = wp; i < s; i += nw) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) v[q] = (lane + 32 * q < n) ? A[(int64_t)i * lda + lane + 32 * q] : 0.0;
    for (int j = lane + 128; j < n; j += 32) Wm[(int64_t)i * ld + j] = A[(int64_t)i * lda + j];
#pragma unroll
    for (int q = 0; q < 4; q++) if (lane + 32 * q < n) Wm[(int64_t)i * ld + lane + 32 * q] = v[q];
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  // reflector of column k (called by the owner warp of column k); returns nothing,
  // publishes tau in tauS[k & 1], writes beta on the diagonal and v below it
  // all row loops run a warp-uniform trip count with a predicated body, so the warp is
  // converged at every shuffle (no WARPSYNC.COLLECTIVE slow path)
  auto reflector = [&](int k) {
    double part = 0.0;
    for (int i0 = k + 1; i0 < s; i0 += 32) {
      const int i = i0 + lane;
      const double x = i < s ? Wm[(int64_t)i * ld + k] : 0.0;
      part = __fma_rn(x, x, part);
    }
    __syncwarp();
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double alpha = Wm[(int64_t)k * ld + k];
    const double xnorm = __dsqrt_rn(part);
    double beta = alpha, tau = 0.0;
    if (xnorm != 0.0) {
      beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, xnorm);
      tau = __ddiv_rn(beta - alpha, beta);
      const double sc = __ddiv_rn(1.0, alpha - beta);
      for (int i0 = k + 1; i0 < s; i0 += 32) {
        const int i = i0 + lane;
        if (i < s) Wm[(int64_t)i * ld + k] *= sc;
      }
    } else if (alpha == 0.0 && lane == 0) {
      report(status, RLHC_ERANKDEF, RLHC_STAGE_HQR, k);
      flag = 1;
    }
    __syncwarp();
    if (lane == 0) { tauS[k & 1] = tau; Wm[(int64_t)k * ld + k] = beta; }
  };
  auto apply = [&](int k, int j, double tau) {
    double acc = 0.0;
    for (int i0 = k + 1; i0 < s; i0 += 32) {
      const int i = i0 + lane;
      if (i < s) acc = __fma_rn(Wm[(int64_t)i * ld + k], Wm[(int64_t)i * ld + j], acc);
    }
    __syncwarp();
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const double tw = tau * (Wm[(int64_t)k * ld + j] + acc);
    __syncwarp();
    if (lane == 0) Wm[(int64_t)k * ld + j] -= tw;
    for (int i0 = k + 1; i0 < s; i0 += 32) {
      const int i = i0 + lane;
      if (i < s) Wm[(int64_t)i * ld + j] = __fma_rn(-Wm[(int64_t)i * ld + k], tw, Wm[(int64_t)i * ld + j]);
    }
    __syncwarp();
  };
  if (wp == 0) reflector(0);
  __syncthreads();
  for (int k = 0; k < n; k++) {
    if (flag) break;
    const double tau = tauS[k & 1];
    const int jn = k + 1;  // next pivot column
    if (jn < n && (jn % nw) == wp) {
      if (tau != 0.0) apply(k, jn, tau);
      reflector(jn);
    }
    if (tau != 0.0)
      for (int j = k + 1 + ((wp - (k + 1)) % nw + nw) % nw; j < n; j += nw)
        if (j != jn) apply(k, j, tau);
    __syncthreads();
  }
  for (int i = wp; i < n; i += nw) {
    const double d = Wm[(int64_t)i * ld + i];
    const bool flip = sgn_ref && ((d < 0.0) != (sgn_ref[(int64_t)i * n + i] < 0.0));
    for (int j = lane; j < n; j += 32) {
      double v = (j >= i) ? Wm[(int64_t)i * ld + j] : 0.0;
      S[(int64_t)i * n + j] = flip ? -v : v;
    }
  }
}

constexpr int HQ_WARPS = 16;

// ------------------------------------------------------------------ register-resident HQR
// For s <= 32*RR, n <= 16*QC the s x n sketch lives in REGISTERS of 16 warps: column j owned
// by warp j mod 16, lane l holds rows l + 32 r (reflector formulas of R#O7), without CTA
// barriers (a barrier per step measured ~3000 cycles/step): step k's reflector is published to shared memory
// (v_k, tau_k) and signalled by mbarrier k.  The owner of column k+1 (another warp) applies
// reflector k to that column first, forms reflector k+1 and publishes it, then applies k to
// its later columns; every other warp applies k to its columns as soon as it is published.
// All reflectors stay in shared memory (n x s doubles), so no slot is reused.
template <int RR, int QC>
struct HqpSmem {
  double v[16 * QC][32 * RR];
  double tau[16 * QC];
  double beta[16 * QC];
  unsigned long long bar[16 * QC];
};

template <int RR, int QC>
RLHC_DEV void hqp_apply(double (&a)[RR][QC], int q, const double (&v)[RR], double tau) {
  double dot = 0.0;
#pragma unroll
  for (int r = 0; r < RR; r++) dot = __fma_rn(v[r], a[r][q], dot);
  for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  const double tw = tau * dot;
#pragma unroll
  for (int r = 0; r < RR; r++) a[r][q] = __fma_rn(-v[r], tw, a[r][q]);
}

template <int RR, int QC>
__global__ void __launch_bounds__(32 * HQ_WARPS)
hqr_pipe_kernel(const double* __restrict__ A, int s, int n, int64_t lda, const double* __restrict__ sgn_ref,
                double* __restrict__ S, unsigned long long* status) {
  extern __shared__ __align__(16) unsigned char hq_raw[];
  HqpSmem<RR, QC>& sm = *reinterpret_cast<HqpSmem<RR, QC>*>(hq_raw);
  const int lane = lane_id(), wp = warp_id();
  double a[RR][QC];
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int q = 0; q < QC; q++) {
      const int i = lane + 32 * r, j = wp + HQ_WARPS * q;
      a[r][q] = (i < s && j < n) ? A[(int64_t)i * lda + j] : 0.0;
    }
  for (int k = threadIdx.x; k < 16 * QC; k += blockDim.x) mbar_init(&sm.bar[k], 32);
  __syncthreads();
  // the warp's last column; it has nothing to do after step last-1
  const int last = wp + HQ_WARPS * ((n - 1 - wp) / HQ_WARPS);
  double v[RR], tau = 0.0;
#pragma unroll
  for (int Q = 0; Q < QC; Q++) {
#pragma unroll 1
    for (int jj = 0; jj < HQ_WARPS; jj++) {
      const int k = Q * HQ_WARPS + jj;  // step k: reflector of column k (owner: warp jj)
      if (k >= n || wp >= n || k > last) break;
      if (k > 0) {
        mbar_wait(&sm.bar[k - 1], 0);
        tau = sm.tau[k - 1];
#pragma unroll
        for (int r = 0; r < RR; r++) v[r] = sm.v[k - 1][lane + 32 * r];
      }
      if (jj == wp) {
        // column k = (wp, Q): reflector k-1 first, then form reflector k and publish it
        if (k > 0 && tau != 0.0) hqp_apply<RR, QC>(a, Q, v, tau);
        double part = 0.0, alpha = 0.0;
#pragma unroll
        for (int r = 0; r < RR; r++) {
          const int i = lane + 32 * r;
          if (i > k && i < s) part = __fma_rn(a[r][Q], a[r][Q], part);
          if (i == k) alpha = a[r][Q];
        }
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        alpha = __shfl_sync(0xffffffffu, alpha, k & 31);
        double beta = alpha, tk = 0.0, sc = 0.0;
        if (part != 0.0) {
          // beta = -sign(alpha) ||(alpha, x)|| (R#O7; sum of squares already formed, so the
          // norm is taken directly rather than through hypot)
          beta = -(alpha >= 0.0 ? 1.0 : -1.0) * __dsqrt_rn(__fma_rn(alpha, alpha, part));
          tk = __ddiv_rn(beta - alpha, beta);
          sc = __ddiv_rn(1.0, alpha - beta);
        } else if (alpha == 0.0 && lane == 0) {
          report(status, RLHC_ERANKDEF, RLHC_STAGE_HQR, k);
        }
#pragma unroll
        for (int r = 0; r < RR; r++) {
          const int i = lane + 32 * r;
          sm.v[k][i] = (i > k) ? a[r][Q] * sc : (i == k ? 1.0 : 0.0);
          if (i == k) a[r][Q] = beta;
        }
        if (lane == 0) {
          sm.tau[k] = tk;
          sm.beta[k] = beta;
        }
        __syncwarp();
        mbar_arrive(&sm.bar[k]);
        // reflector k-1 on this warp's later columns
        if (k > 0 && tau != 0.0) {
#pragma unroll
          for (int q = Q + 1; q < QC; q++)
            if (wp + HQ_WARPS * q < n) hqp_apply<RR, QC>(a, q, v, tau);
        }
      } else if (k > 0 && tau != 0.0) {
        // reflector k-1 on this warp's columns >= k (column (wp, Q) if wp > jj, and later ones)
#pragma unroll
        for (int q = Q; q < QC; q++)
          if ((q > Q || wp > jj) && wp + HQ_WARPS * q < n) hqp_apply<RR, QC>(a, q, v, tau);
      }
    }
  }
  __syncthreads();
  // R = upper n x n part (diag = beta_k), sign-aligned with sgn_ref (R#7)
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int q = 0; q < QC; q++) {
      const int i = lane + 32 * r, j = wp + HQ_WARPS * q;
      if (i < n && j < n) {
        double val = (j >= i) ? a[r][q] : 0.0;
        if (sgn_ref && ((sm.beta[i] < 0.0) != (sgn_ref[(int64_t)i * n + i] < 0.0))) val = -val;
        S[(int64_t)i * n + j] = val;
      }
    }
}

// ------------------------------------------------------------------ blocked Householder R
// For sketches that do not fit one CTA's registers (cfg3: 256 x 128, cfg4: 1024 x 512), the
// LAPACK dgeqrf structure on a row-major working copy Wk (s x n, ld n):
//   for each panel of HB columns [j0, j0+HB):
//     hqr_panel_kernel  (1 CTA, 512 threads, lane = row, the (s-j0) x HB panel in registers):
//       dgeqr2 on the panel (same reflector formulas as above, R#O7); V stays in place below
//       the diagonal, R on/above it.  The compact-WY factor T (H_0..H_{HB-1} = I - V T V^T)
//       is built from the SAME block reductions: at step k the reduction that forms
//       w_c = v_k^T A(:, c) for the panel columns c > k also yields z_j = V(:, j)^T v_k for
//       j < k, and T(0:k, k) = -tau_k T(0:k, 0:k) z.
//     hqr_trail_kernel  (1 CTA per 16 trailing columns): Y = V^T A_blk (DMMA, rows split
//       over warps), Z = T^T Y, A_blk -= V Z (DMMA).
// The blocked order only re-associates the reflector applications (R agrees with dgeqr2 to
// rounding; HQR output is tolerance-checked).
// one transpose-reduce round: CNT live values, exchange half of them across lane bit O
template <int CNT, int O, int HB>
RLHC_DEV void hb_round(double (&v)[HB], int lane, int& base) {
  if constexpr (CNT > 1 && O >= 2) {
    const bool hi = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < CNT / 2; i++) {
      const double keep = hi ? v[i + CNT / 2] : v[i];
      const double send = hi ? v[i] : v[i + CNT / 2];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    base += hi ? CNT / 2 : 0;
    hb_round<CNT / 2, O / 2, HB>(v, lane, base);
  } else {
    // the single live value: reduce over the remaining lane bits O .. 1
#pragma unroll
    for (int o = O; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  }
}

// Block sum of HB values over 16 warps; every thread gets the totals.  Warp stage:
// transpose-reduce (2 HB - 1 shuffles instead of 5 HB).
template <int HB>
RLHC_DEV void hb_block_sum(double (&y)[HB], double (&red)[16][HB + 1], double (&tot)[HB]) {
  static_assert(HB == 16 || HB == 8, "HB");
  const int lane = lane_id(), wp = warp_id();
  int base = 0;
  hb_round<HB, 16, HB>(y, lane, base);
  constexpr int LOG = HB == 16 ? 4 : 3;
  if ((lane & ((32 >> LOG) - 1)) == 0) red[wp][base] = y[0];
  __syncthreads();
  if (threadIdx.x < HB) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < 16; w++) sum += red[w][threadIdx.x];
    tot[threadIdx.x] = sum;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < HB; i++) y[i] = tot[i];
}

RLHC_DEV double hb_warp_sum(double x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int RPT, int HB>
__global__ void __launch_bounds__(512)
hqr_panel_kernel(double* __restrict__ Wk, int s, int n, int j0, double* __restrict__ Tg,
                 unsigned long long* status) {
  __shared__ double red[16][HB + 1];
  __shared__ double tot[HB];
  __shared__ double Ts[HB][HB + 1];
  __shared__ double bc[2];
  const int tid = threadIdx.x, lane = lane_id(), wp = warp_id();
  const int r = s - j0, nb = min(HB, n - j0);
  double x[RPT][HB];
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int li = tid + 512 * q;
    const double* p = Wk + (int64_t)(j0 + li) * n + j0;
#pragma unroll
    for (int c = 0; c < HB; c++) x[q][c] = (li < r && c < nb) ? p[c] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < HB; k++) {
    if (k >= nb) break;
    // (1) sigma = ||A(k+1:, k)||^2, alpha = A(k, k)
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      const int li = tid + 512 * q;
      if (li > k && li < r) part = __fma_rn(x[q][k], x[q][k], part);
    }
    part = hb_warp_sum(part);
    if (lane == 0) red[wp][0] = part;
    if (tid == k) bc[0] = x[0][k];
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < 16; w++) sum += red[w][0];
      tot[0] = sum;
    }
    __syncthreads();
    const double alpha = bc[0], xnorm = __dsqrt_rn(tot[0]);
    double beta = alpha, tau = 0.0, sc = 0.0;
    if (xnorm != 0.0) {
      beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, xnorm);
      tau = __ddiv_rn(beta - alpha, beta);
      sc = __ddiv_rn(1.0, alpha - beta);
    } else if (alpha == 0.0 && tid == 0) {
      report(status, RLHC_ERANKDEF, RLHC_STAGE_HQR, j0 + k);
    }
    // (2) v (1 at row k), R(k, k) = beta; y_c = v^T A(:, c) for every panel column c != k
    double vv[RPT], y[HB];
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      const int li = tid + 512 * q;
      vv[q] = (li > k && li < r) ? x[q][k] * sc : (li == k ? 1.0 : 0.0);
      if (li > k) x[q][k] = vv[q];
      if (li == k) x[q][k] = beta;
    }
#pragma unroll
    for (int c = 0; c < HB; c++) {
      double acc = 0.0;
      if (c != k) {
#pragma unroll
        for (int q = 0; q < RPT; q++) acc = __fma_rn(vv[q], x[q][c], acc);
      }
      y[c] = acc;
    }
    hb_block_sum<HB>(y, red, tot);
    // (3) trailing panel columns; (4) column k of T from z = y[0:k]
#pragma unroll
    for (int c = k + 1; c < HB; c++) {
      const double tw = tau * y[c];
#pragma unroll
      for (int q = 0; q < RPT; q++) x[q][c] = __fma_rn(-vv[q], tw, x[q][c]);
    }
    if (tid < k) {
      double acc = 0.0;
      for (int p = tid; p < k; p++) acc = __fma_rn(Ts[tid][p], tot[p], acc);  // tot == y (smem copy)
      Ts[tid][k] = -tau * acc;
    } else if (tid == k) {
      Ts[k][k] = tau;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int li = tid + 512 * q;
    double* p = Wk + (int64_t)(j0 + li) * n + j0;
    if (li < r)
#pragma unroll
      for (int c = 0; c < HB; c++)
        if (c < nb) p[c] = x[q][c];
  }
  for (int e = tid; e < HB * HB; e += blockDim.x) {
    const int i = e / HB, j = e - i * HB;
    Tg[e] = (i < nb && j < nb && j >= i) ? Ts[i][j] : 0.0;
  }
}

// V(li, p) of the current panel (unit lower trapezoid stored below the diagonal of Wk)
RLHC_DEV double hb_v(const double* Wk, int n, int j0, int r, int nb, int li, int p) {
  if (li >= r || p >= nb || li < p) return 0.0;
  return li == p ? 1.0 : Wk[(int64_t)(j0 + li) * n + j0 + p];
}

// A(j0:, c0:c0+16) -= V (T^T (V^T A)) for one 16-column block; 8 warps.
template <int HB>
__global__ void __launch_bounds__(256)
hqr_trail_kernel(double* __restrict__ Wk, int s, int n, int j0, const double* __restrict__ Tg) {
  static_assert(HB == 16 || HB == 8, "panel width");
  constexpr int MT = HB / 8;  // m-tiles of Y (rows p)
  __shared__ double Yw[8][HB][17];
  __shared__ double Zs[HB][17];
  const int lane = lane_id(), wp = warp_id(), g = lane >> 2, t = lane & 3;
  const int r = s - j0, nb = min(HB, n - j0);
  const int c0 = j0 + nb + blockIdx.x * 16;
  // pass 1: Y = V^T A_blk, k = rows (4 per DMMA), split over warps
  double acc[MT][2][2];
#pragma unroll
  for (int i = 0; i < MT; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 4 * wp; k0 < r; k0 += 32) {
    const int li = k0 + t;
    double a[MT], b[2];
#pragma unroll
    for (int mt = 0; mt < MT; mt++) a[mt] = hb_v(Wk, n, j0, r, nb, li, mt * 8 + g);
#pragma unroll
    for (int nt = 0; nt < 2; nt++) {
      const int c = c0 + nt * 8 + g;
      b[nt] = (li < r && c < n) ? Wk[(int64_t)(j0 + li) * n + c] : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int nt = 0; nt < 2; nt++) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < MT; mt++)
#pragma unroll
    for (int nt = 0; nt < 2; nt++) {
      Yw[wp][mt * 8 + g][nt * 8 + 2 * t] = acc[mt][nt][0];
      Yw[wp][mt * 8 + g][nt * 8 + 2 * t + 1] = acc[mt][nt][1];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < HB * 16; e += blockDim.x) {
    const int p = e >> 4, c = e & 15;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < 8; w++) sum += Yw[w][p][c];
    Yw[0][p][c] = sum;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < HB * 16; e += blockDim.x) {
    const int p = e >> 4, c = e & 15;
    double z = 0.0;
    for (int q = 0; q <= p; q++) z = __fma_rn(Tg[q * HB + p], Yw[0][q][c], z);  // (T^T Y)(p, c)
    Zs[p][c] = z;
  }
  __syncthreads();
  // pass 2: A_blk -= V Z, m = rows (8 per tile), k = p
  for (int m0 = 8 * wp; m0 < r; m0 += 64) {
    const int li = m0 + g;
    double d[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int c = c0 + nt * 8 + 2 * t + e;
        d[nt][e] = (li < r && c < n) ? Wk[(int64_t)(j0 + li) * n + c] : 0.0;
      }
#pragma unroll
    for (int kk = 0; kk < HB / 4; kk++) {
      const double a = -hb_v(Wk, n, j0, r, nb, li, 4 * kk + t);
#pragma unroll
      for (int nt = 0; nt < 2; nt++) dmma(d[nt][0], d[nt][1], a, Zs[4 * kk + t][nt * 8 + g]);
    }
#pragma unroll
    for (int nt = 0; nt < 2; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int c = c0 + nt * 8 + 2 * t + e;
        if (li < r && c < n) Wk[(int64_t)(j0 + li) * n + c] = d[nt][e];
      }
  }
}

__global__ void hqr_copy_kernel(const double* __restrict__ A, int s, int n, int64_t lda, double* __restrict__ Wk) {
  const int64_t total = (int64_t)s * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    Wk[e] = A[i * lda + j];
  }
}

// S = upper n x n of Wk, rows sign-aligned with sgn_ref (R#7)
__global__ void hqr_finish_kernel(const double* __restrict__ Wk, int n, const double* __restrict__ sgn_ref,
                                  double* __restrict__ S) {
  const int i = blockIdx.x;
  const double d = Wk[(int64_t)i * n + i];
  const bool flip = sgn_ref && ((d < 0.0) != (sgn_ref[(int64_t)i * n + i] < 0.0));
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double v = (j >= i) ? Wk[(int64_t)i * n + j] : 0.0;
    S[(int64_t)i * n + j] = flip ? -v : v;
  }
}

template <int RPT, int HB>
static void run_hqr_blocked(const double* A, int s, int n, int64_t lda, const double* sgn_ref, double* S,
                            double* Wk, double* Tg, unsigned long long* status, cudaStream_t st) {
  note_launch();
  hqr_copy_kernel<<<kSMs, 256, 0, st>>>(A, s, n, lda, Wk);
  for (int j0 = 0; j0 < n; j0 += HB) {
    note_launch();
    hqr_panel_kernel<RPT, HB><<<1, 512, 0, st>>>(Wk, s, n, j0, Tg, status);
    const int rest = n - j0 - HB;
    if (rest > 0) {
      note_launch();
      hqr_trail_kernel<HB><<<ceil_div(rest, 16), 256, 0, st>>>(Wk, s, n, j0, Tg);
    }
  }
  note_launch();
  hqr_finish_kernel<<<n, 128, 0, st>>>(Wk, n, sgn_ref, S);
}

size_t hqr_ws_bytes(int s, int n) {
  return std::max((size_t)s * (n + 1), (size_t)s * n + 16 * 16) * sizeof(double);
}

cudaError_t launch_hqr(const double* A, int s, int n, int64_t lda, const double* sgn_ref, double* S, double* work,
                       unsigned long long* status, cudaStream_t st) {
  const size_t need = hqr_ws_bytes(s, n);
  const int threads = n >= 512 ? 1024 : 512;
#define HQR_REG(RR, QC)                                                                            \
  if (s <= 32 * RR && n <= HQ_WARPS * QC) {                                                        \
    constexpr int smem = (int)sizeof(HqpSmem<RR, QC>);                                             \
    static DevFlags attr;                                                                          \
    if (cudaError_t e_ = smem_attr(attr, hqr_pipe_kernel<RR, QC>, smem)) return e_;                \
    note_launch();                                                                                 \
    hqr_pipe_kernel<RR, QC><<<1, 32 * HQ_WARPS, smem, st>>>(A, s, n, lda, sgn_ref, S, status);     \
    return cudaGetLastError();                                                                     \
  }
  HQR_REG(1, 1)
  HQR_REG(2, 2)
  HQR_REG(4, 4)
  HQR_REG(8, 4)
  HQR_REG(4, 8)
#undef HQR_REG
  // blocked path (Wk = work[0 : s*n), T after it)
  if (s <= 512) { run_hqr_blocked<1, 16>(A, s, n, lda, sgn_ref, S, work, work + (size_t)s * n, status, st); return cudaGetLastError(); }
  if (s <= 1024) { run_hqr_blocked<2, 16>(A, s, n, lda, sgn_ref, S, work, work + (size_t)s * n, status, st); return cudaGetLastError(); }
  if (s <= 2048) { run_hqr_blocked<4, 8>(A, s, n, lda, sgn_ref, S, work, work + (size_t)s * n, status, st); return cudaGetLastError(); }
  if (need <= 200 * 1024) {
    if (need > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(hqr2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
      if (e) return e;
    }
    note_launch();
    hqr2_kernel<true><<<1, threads, need, st>>>(A, s, n, lda, sgn_ref, S, work, status);
  } else {
    note_launch();
    hqr2_kernel<false><<<1, 1024, 0, st>>>(A, s, n, lda, sgn_ref, S, work, status);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Cholesky
// Upper R with R^T R = G, right-looking on a working copy (row stride n+1): per
// step k one thread forms r_kk (a pivot <= 0 or non-finite -> EBREAKDOWN(stage, k), SPEC
// S:55, and the factorization stops), row k is divided by r_kk, and warp (j mod NW)
// updates column j of the trailing matrix.
template <bool SMEM>
__global__ void __launch_bounds__(256)
chol2_kernel(const double* __restrict__ G, int n, double* __restrict__ R, double* __restrict__ work, int stage,
             unsigned long long* status) {
  extern __shared__ double dsm[];
  __shared__ int flag;
  __shared__ double rkk_s;
  const int ld = n + 1;
  double* C = SMEM ? dsm : work;
  const int lane = lane_id(), wp = warp_id(), nw = blockDim.x >> 5;
  for (int i = wp; i < n; i += nw) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) v[q] = (lane + 32 * q < n) ? G[(int64_t)i * n + lane + 32 * q] : 0.0;
    for (int j = lane + 128; j < n; j += 32) C[(int64_t)i * ld + j] = G[(int64_t)i * n + j];
#pragma unroll
    for (int q = 0; q < 4; q++) if (lane + 32 * q < n) C[(int64_t)i * ld + lane + 32 * q] = v[q];
  }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int k = 0; k < n; k++) {
    if (threadIdx.x == 0) {
      const double d = C[(int64_t)k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) { report(status, RLHC_EBREAKDOWN, stage, k); flag = 1; }
      else { rkk_s = __dsqrt_rn(d); C[(int64_t)k * ld + k] = rkk_s; }
    }
    __syncthreads();
    if (flag) break;
    const double rkk = rkk_s;
    for (int j = k + 1 + threadIdx.x; j < n; j += blockDim.x)
      C[(int64_t)k * ld + j] = __ddiv_rn(C[(int64_t)k * ld + j], rkk);
    __syncthreads();
    for (int j = k + 1 + wp; j < n; j += nw) {
      const double ckj = C[(int64_t)k * ld + j];
      for (int i = k + 1 + lane; i <= j; i += 32)
        C[(int64_t)i * ld + j] = __fma_rn(-C[(int64_t)k * ld + i], ckj, C[(int64_t)i * ld + j]);
    }
    __syncthreads();
  }
  for (int i = wp; i < n; i += nw)
    for (int j = lane; j < n; j += 32) R[(int64_t)i * n + j] = (j >= i) ? C[(int64_t)i * ld + j] : 0.0;
}

// ------------------------------------------------------------------ pipelined Cholesky
// n <= 128: G (symmetric) in REGISTERS of 16 warps, column j owned by warp j mod 16, lane l
// holds rows l + 32 r.  Right-looking, no CTA barriers: the owner of column k applies step
// k-1 to it, takes d = a_kk (d <= 0 or non-finite -> EBREAKDOWN(stage, koff + k), SPEC
// S:55), r_kk = sqrt(d), publishes the column l_k = a(:, k) / r_kk (rows > k; r_kk at k) and
// 1/r_kk through shared memory + mbarrier k, then applies step k-1 to its later columns;
// every other warp applies a(:, j) -= l_k * l_k(j) to its columns j > k as soon as l_k is
// published.  R(k, j) = l_k(j) for j >= k; 1/diag(R) is emitted for the substitution passes.
template <int RR, int QC>
struct CholSmem {
  double l[16 * QC][32 * RR];
  double rinv[16 * QC];
  unsigned long long bar[16 * QC];
};

template <int RR, int QC>
__global__ void __launch_bounds__(512)
chol_pipe_kernel(const double* __restrict__ G, int64_t ldg, int n, double* __restrict__ R, int64_t ldr,
                 double* __restrict__ rdiag, int stage, int koff, unsigned long long* status) {
  extern __shared__ __align__(16) unsigned char ch_raw[];
  CholSmem<RR, QC>& sm = *reinterpret_cast<CholSmem<RR, QC>*>(ch_raw);
  const int lane = lane_id(), wp = warp_id();
  double a[RR][QC];
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int q = 0; q < QC; q++) {
      const int i = lane + 32 * r, j = wp + 16 * q;
      a[r][q] = (i < n && j < n) ? G[(int64_t)i * ldg + j] : 0.0;
    }
  for (int k = threadIdx.x; k < 16 * QC; k += blockDim.x) mbar_init(&sm.bar[k], 32);
  __syncthreads();
  const int last = wp < n ? wp + 16 * ((n - 1 - wp) / 16) : -1;
  double lk[RR];
#pragma unroll
  for (int Q = 0; Q < QC; Q++) {
#pragma unroll 1
    for (int jj = 0; jj < 16; jj++) {
      const int k = Q * 16 + jj;  // step k: column k (owner warp jj)
      if (k >= n || k > last) break;
      if (k > 0) {
        mbar_wait(&sm.bar[k - 1], 0);
#pragma unroll
        for (int r = 0; r < RR; r++) lk[r] = sm.l[k - 1][lane + 32 * r];
      }
      // a(:, j) -= l_{k-1} * l_{k-1}(j) for this warp's columns j in [q_lo, QC) (j >= k)
      auto update = [&](int q) {
        const double s = sm.l[k - 1][wp + 16 * q];
#pragma unroll
        for (int r = 0; r < RR; r++) a[r][q] = __fma_rn(-lk[r], s, a[r][q]);
      };
      if (jj == wp) {
        if (k > 0) update(Q);
        double d = 0.0;
#pragma unroll
        for (int r = 0; r < RR; r++) d = (lane + 32 * r == k) ? a[r][Q] : d;
        d = __shfl_sync(0xffffffffu, d, k & 31);
        if (lane == 0 && (!(d > 0.0) || !isfinite(d))) report(status, RLHC_EBREAKDOWN, stage, koff + k);
        const double rk = __dsqrt_rn(d), ri = __drcp_rn(rk);
#pragma unroll
        for (int r = 0; r < RR; r++) {
          const int i = lane + 32 * r;
          sm.l[k][i] = (i > k) ? __dmul_rn(a[r][Q], ri) : (i == k ? rk : 0.0);
        }
        if (lane == 0) sm.rinv[k] = ri;
        __syncwarp();
        mbar_arrive(&sm.bar[k]);
        if (k > 0) {
#pragma unroll
          for (int q = Q + 1; q < QC; q++)
            if (wp + 16 * q < n) update(q);
        }
      } else if (k > 0) {
#pragma unroll
        for (int q = Q; q < QC; q++)
          if ((q > Q || wp > jj) && wp + 16 * q < n) update(q);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int k = e / n, j = e - k * n;
    R[(int64_t)k * ldr + j] = (j >= k) ? sm.l[k][j] : 0.0;
  }
  if (rdiag)
    for (int k = threadIdx.x; k < n; k += blockDim.x) rdiag[k] = sm.rinv[k];
}

template <int RR, int QC>
static cudaError_t run_chol_pipe(const double* G, int64_t ldg, int n, double* R, int64_t ldr, double* rdiag, int stage,
                                 int koff, unsigned long long* status, cudaStream_t st) {
  constexpr int smem = (int)sizeof(CholSmem<RR, QC>);
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, chol_pipe_kernel<RR, QC>, smem)) return e;
  note_launch();
  chol_pipe_kernel<RR, QC><<<1, 512, smem, st>>>(G, ldg, n, R, ldr, rdiag, stage, koff, status);
  return cudaGetLastError();
}

static cudaError_t launch_chol_pipe(const double* G, int64_t ldg, int n, double* R, int64_t ldr, double* rdiag,
                                    int stage, int koff, unsigned long long* status, cudaStream_t st) {
  if (n <= 32) return run_chol_pipe<1, 2>(G, ldg, n, R, ldr, rdiag, stage, koff, status, st);
  if (n <= 64) return run_chol_pipe<2, 4>(G, ldg, n, R, ldr, rdiag, stage, koff, status, st);
  return run_chol_pipe<4, 8>(G, ldg, n, R, ldr, rdiag, stage, koff, status, st);
}


__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int rows, int cols, double* __restrict__ B,
                                 int64_t ldb) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? A[(int64_t)r * lda + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) B[(int64_t)c * ldb + r] = tile[threadIdx.x][i];
  }
}

__global__ void zero_lower_kernel(double* R, int n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x)
    if (e / n > e % n) R[e] = 0.0;
}

// n > 128: 64-column blocks.  Per block: the 64 x 64 diagonal block by chol_pipe_kernel,
// R12^T = C21 R_pp^{-1} (rowsolve on the rows below), R12 = its transpose, and the trailing
// update C22 -= R12^T R12 on DMMA (gemm_update).  `work` holds the working copy of G (n x n)
// and the R12^T scratch (n x 64).
static cudaError_t launch_chol_big(const double* G, int n, double* R, double* work, int stage,
                                   unsigned long long* status, cudaStream_t st) {
  double* Cw = work;
  double* R12t = work + (size_t)n * n;
  double* rd = R12t + (size_t)n * 64;
  cudaError_t e = cudaMemcpyAsync(Cw, G, (size_t)n * n * 8, cudaMemcpyDeviceToDevice, st);
  if (e) return e;
  e = cudaMemsetAsync(R, 0, (size_t)n * n * 8, st);
  if (e) return e;
  for (int p0 = 0; p0 < n; p0 += 64) {
    const int w = std::min(64, n - p0);
    e = launch_chol_pipe(Cw + (size_t)p0 * n + p0, n, w, R + (size_t)p0 * n + p0, n, nullptr, stage, p0, status, st);
    if (e) return e;
    const int N = n - p0 - w;
    if (N <= 0) break;
    e = launch_rdiag(R + (size_t)p0 * n + p0, w, n, rd, stage, status, st);
    if (e) return e;
    // R12^T (N x w) = C21 (rows below the block) * R_pp^{-1}
    e = launch_trsm_blocked(Cw + (size_t)(p0 + w) * n + p0, n, N, w, w, R + (size_t)p0 * n + p0, n, rd, R12t, 64, st);
    if (e) return e;
    note_launch();
    transpose_kernel<<<dim3(ceil_div(w, 32), ceil_div(N, 32)), dim3(32, 8), 0, st>>>(R12t, 64, N, w,
                                                                                     R + (size_t)p0 * n + p0 + w, n);
    e = cudaGetLastError();
    if (e) return e;
    // C22 -= R12^T R12
    e = launch_gemm_update(Cw + (size_t)(p0 + w) * n + p0 + w, n, Cw + (size_t)(p0 + w) * n + p0 + w, n, R12t, 64,
                           R + (size_t)p0 * n + p0 + w, n, N, w, N, st);
    if (e) return e;
  }
  return cudaSuccess;
}

size_t chol_ws_bytes(int n) {
  return std::max((size_t)n * (n + 1) * sizeof(double), ((size_t)n * n + (size_t)n * 64 + 64) * sizeof(double));
}

cudaError_t launch_chol(const double* G, int n, double* R, double* work, int stage, unsigned long long* status,
                        cudaStream_t st, double* rdiag) {
  const size_t need = (size_t)n * (n + 1) * sizeof(double);
  if (n <= 128) return launch_chol_pipe(G, n, n, R, n, rdiag, stage, 0, status, st);
  if (work) return launch_chol_big(G, n, R, work, stage, status, st);
  if (need <= 200 * 1024) {
    if (need > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(chol2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
      if (e) return e;
    }
    note_launch();
    chol2_kernel<true><<<1, 256, need, st>>>(G, n, R, work, stage, status);
  } else {
    if (!work) return cudaErrorInvalidValue;
    note_launch();
    chol2_kernel<false><<<1, 256, 0, st>>>(G, n, R, work, stage, status);
  }
  return cudaGetLastError();
}

}  // namespace rlhc
