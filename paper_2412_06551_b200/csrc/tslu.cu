// tslu.cu -- tournament-pivoted tall-skinny LU "PX = LU"
// under the pivot contract of DESIGN.md R#3-R#5 (tslu over column panels).
//
// One select CTA holds R = 32*RS candidate rows of a W-wide panel in REGISTERS,
// column-owned (select.cuh): warp q holds columns [q*W/NW, (q+1)*W/NW) of every candidate
// row and runs GEPP as a producer/consumer pipeline over per-step mbarriers -- no CTA-wide
// barrier inside the elimination.
#include <climits>

#include "common.cuh"
#include "kernels.cuh"
#include "select.cuh"

namespace rlhc {

// Leaf select: leaf = global row block [leaf*R, leaf*R + R) of the LOCAL rows
// (global id = row0 + local row).  src: current values (X for the first panel, the
// trailing matrix afterwards), panel columns [p0, p0 + w).  Output level slot = leaf.
template <int W, int NW, int RS>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_leaf_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                 const uint8_t* __restrict__ chosen, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals, RootOut root, unsigned long long* finite_status) {
  constexpr int R = 32 * RS, CW = W / NW;
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelSmem<W, NW, RS>& sm = *reinterpret_cast<SelSmem<W, NW, RS>*>(sel_raw);
  sel_init(sm, root.U, root.n);
  const int lane = lane_id(), wp = warp_id();
  double a[RS][CW];
  int gid[RS];
  unsigned act = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int64_t r = (int64_t)blockIdx.x * R + s * 32 + lane;
    const bool ok = r < rows && !(chosen && chosen[r]);
    act |= (ok ? 1u : 0u) << s;
    gid[s] = (int)(row0 + r);
    const double* p = src + r * lds + p0 + wp;
#pragma unroll
    for (int c = 0; c < CW; c++) a[s][c] = (ok && wp + NW * c < w) ? p[NW * c] : 0.0;
  }
  // single-panel pipelines fold the input check (check_finite_kernel's semantics: the
  // smallest non-finite element index i*n + j wins) into this pass over X
  if (finite_status) {
#pragma unroll
    for (int s = 0; s < RS; s++)
#pragma unroll
      for (int c = 0; c < CW; c++)
        if (!isfinite(a[s][c]))
          report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT,
                 ((int64_t)blockIdx.x * R + s * 32 + lane) * w + wp + NW * c);
  }
  const int steps = gepp_select<W, NW, RS>(a, act, gid, w, sm);
  if (root.U) sel_root_finish(sm, steps, w, root);
  int* oi = out_ids + (size_t)blockIdx.x * W;
  double* ov = out_vals + (size_t)blockIdx.x * W * W;
  if (threadIdx.x == 0) out_cnt[blockIdx.x] = steps;
  for (int e = threadIdx.x; e < W; e += blockDim.x) oi[e] = e < steps ? sm.out_id[e] : -1;
  for (int idx = threadIdx.x; idx < steps * w; idx += blockDim.x) {
    int e = idx / w, c = idx - e * w;
    int64_t rr = (int64_t)blockIdx.x * R + sm.out_src[e];
    ov[e * W + c] = src[rr * lds + p0 + c];
  }
}

// Node select: node = children [node*arity, node*arity + arity) of the level below;
// candidate index q -> child (q / w), entry (q % w).  Values are the stored current
// panel values of the candidates (not the eliminated ones).
template <int W, int NW, int RS>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_node_kernel(const int* __restrict__ in_ids, const int* __restrict__ in_cnt, const double* __restrict__ in_vals,
                 int nslots_in, int arity, int w, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals, RootOut root) {
  constexpr int CW = W / NW;
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelSmem<W, NW, RS>& sm = *reinterpret_cast<SelSmem<W, NW, RS>*>(sel_raw);
  sel_init(sm, root.U, root.n);
  const int lane = lane_id(), wp = warp_id();
  const int c0 = blockIdx.x * arity;
  double a[RS][CW];
  int gid[RS];
  unsigned act = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int qi = s * 32 + lane;
    const int ci = qi / w, e = qi - ci * w;
    const int child = c0 + ci;
    const bool ok = ci < arity && child < nslots_in && e < in_cnt[child < nslots_in ? child : 0];
    act |= (ok ? 1u : 0u) << s;
    const int slot = child * W + e;
    gid[s] = ok ? in_ids[slot] : INT_MAX;
    const double* p = in_vals + (size_t)(ok ? slot : 0) * W + wp;
#pragma unroll
    for (int c = 0; c < CW; c++) a[s][c] = (ok && wp + NW * c < w) ? p[NW * c] : 0.0;
  }
  const int steps = gepp_select<W, NW, RS>(a, act, gid, w, sm);
  if (root.U) sel_root_finish(sm, steps, w, root);
  int* oi = out_ids + (size_t)blockIdx.x * W;
  double* ov = out_vals + (size_t)blockIdx.x * W * W;
  if (threadIdx.x == 0) out_cnt[blockIdx.x] = steps;
  for (int q = threadIdx.x; q < W; q += blockDim.x) oi[q] = q < steps ? sm.out_id[q] : -1;
  for (int idx = threadIdx.x; idx < steps * w; idx += blockDim.x) {
    int q = idx / w, c = idx - q * w;
    const int qi = sm.out_src[q];
    const int ci = qi / w, e = qi - ci * w;
    ov[q * W + c] = in_vals[(size_t)((c0 + ci) * W + e) * W + c];
  }
}

// Panel factor (single CTA): the root's w winners become pivots p0..p0+w-1.  Their
// current rows (src, columns p0..n-1) are eliminated among themselves in pivot order
// -- the same fma chain as in the select -- giving U rows p0..p0+w-1.
//  phase A: the w x w panel block in shared memory, one barrier per pivot;
//  phase B: each trailing column j >= p0+w independently (thread per column).
// Also writes piv[p0..), chosen[] of local pivot rows, and a zero root pivot as
// ERANKDEF(LU, k).
__global__ void __launch_bounds__(512)
tslu_panel_factor_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                         int n, const int* __restrict__ root_ids, const int* __restrict__ root_cnt, double* __restrict__ U,
                         int64_t* __restrict__ piv, uint8_t* __restrict__ chosen, double* __restrict__ lpanel,
                         unsigned long long* status, int packed) {
  __shared__ double P[64][65];
  __shared__ int ids[64];
  __shared__ int64_t srow[64];  // row of src holding pivot t (packed: row t)
  const int tid = threadIdx.x;
  if (tid == 0 && root_cnt[0] < w) report(status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + root_cnt[0]);
  for (int t = tid; t < w; t += blockDim.x) {
    int g = root_ids[t];
    ids[t] = g < 0 ? (int)row0 : g;  // defensive: a short root reports ERANKDEF above
    piv[p0 + t] = g;
    int64_t lr = (int64_t)ids[t] - row0;
    if (chosen && lr >= 0 && lr < rows) chosen[lr] = 1;
    srow[t] = packed ? t : lr;
  }
  __syncthreads();
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    int t = idx / w, c = idx - t * w;
    P[t][c] = src[srow[t] * lds + p0 + c];
  }
  __syncthreads();
  // phase A: right-looking elimination of the w x w block (P[t][t'] <- multiplier for
  // t' < t).  Thread (c = tid & 63, t0 = tid >> 6) owns column c of rows t0, t0+8, ...;
  // every owner recomputes the row multiplier itself (same IEEE ops -> same bits).
  const int c = tid & 63, t0 = tid >> 6;
  for (int k = 0; k < w; k++) {
    const double ukk = P[k][k];
    if (tid == 0 && ukk == 0.0) report(status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + k);
    const double r = __ddiv_rn(1.0, ukk);
    double lv[8], nv[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int t = t0 + 8 * i;
      lv[i] = (t > k && t < w) ? __dmul_rn(P[t][k], r) : 0.0;
      nv[i] = (t > k && t < w && c > k && c < w) ? __fma_rn(-lv[i], P[k][c], P[t][c]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int t = t0 + 8 * i;
      if (t > k && t < w) {
        if (c == k) P[t][k] = lv[i];
        else if (c > k && c < w) P[t][c] = nv[i];
      }
    }
    __syncthreads();
  }
  // U panel block and multipliers of the panel block
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    int t = idx / w, c = idx - t * w;
    if (c >= t) U[(int64_t)(p0 + t) * n + p0 + c] = P[t][c];
    if (lpanel) lpanel[t * 64 + c] = (c < t) ? P[t][c] : (c == t ? 1.0 : 0.0);
  }
  // phase B: trailing columns
  for (int j = p0 + w + tid; j < n; j += blockDim.x) {
    double u[64];
#pragma unroll
    for (int t = 0; t < 64; t++) {
      if (t < w) {
        double v = src[srow[t] * lds + j];
#pragma unroll
        for (int tp = 0; tp < 64; tp++)
          if (tp < t) v = __fma_rn(-P[t][tp], u[tp], v);
        u[t] = v;
        U[(int64_t)(p0 + t) * n + j] = v;
      }
    }
  }
}

// Fixed-up L11 rows: after the pivot rows' X rows were run through the substitution
// (giving their multipliers in columns < k), set the unit diagonal and zero the rest.
__global__ void l11_fixup_kernel(double* L11, int n) {
  int k = blockIdx.x;
  for (int j = k + threadIdx.x; j < n; j += blockDim.x) L11[(int64_t)k * n + j] = (j == k) ? 1.0 : 0.0;
}

__global__ void gather_rows_kernel(const double* __restrict__ src, int64_t lds, const int64_t* __restrict__ ids,
                                   int64_t row0, int cnt, int ncols, double* __restrict__ dst, int64_t ldd) {
  int r = blockIdx.x;
  if (r >= cnt) return;
  const double* s = src + (ids[r] - row0) * lds;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) dst[(int64_t)r * ldd + c] = s[c];
}

__global__ void pivpos_kernel(const int64_t* __restrict__ piv, int n, int64_t row0, int64_t rows, int* __restrict__ pivpos) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    int64_t lr = piv[k] - row0;
    if (lr >= 0 && lr < rows) pivpos[lr] = k;
  }
}

// ------------------------------------------------------------------ host side
int select_rows(int W) { return W == 64 ? 256 : 512; }
// (W, NW, RS): W=64 -> 8 warps x 8 cols, 256 rows; W=32 -> 8 x 4, 512 rows; W=16 -> 8 x 2, 512 rows

template <int W, int NW, int RS>
static cudaError_t run_leaf(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                            const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st,
                            const RootOut& root, unsigned long long* finite_status) {
  int nleaves = (int)ceil_div<int64_t>(rows, 32 * RS);
  constexpr int smem = (int)sizeof(SelSmem<W, NW, RS>);
  static bool attr = false;  // once per instantiation (idempotent, so a race is harmless)
  if (!attr) {
    cudaFuncSetAttribute(tslu_leaf_kernel<W, NW, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tslu_node_kernel<W, NW, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  note_launch(); tslu_leaf_kernel<W, NW, RS><<<nleaves, 32 * NW, smem, st>>>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals,
                                                                            root, finite_status);
  return cudaGetLastError();
}
template <int W, int NW, int RS>
static cudaError_t run_node(const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity, int w,
                            int* ids, int* cnt, double* vals, cudaStream_t st, const RootOut& root) {
  int nout = ceil_div(nin, arity);
  constexpr int smem = (int)sizeof(SelSmem<W, NW, RS>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tslu_leaf_kernel<W, NW, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tslu_node_kernel<W, NW, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  note_launch(); tslu_node_kernel<W, NW, RS><<<nout, 32 * NW, smem, st>>>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt,
                                                                            vals, root);
  return cudaGetLastError();
}

cudaError_t launch_tslu_leaf(int W, const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                             const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st,
                             const RootOut* rootp, unsigned long long* finite_status) {
  const RootOut root = rootp ? *rootp : RootOut{};
  switch (W) {
    case 16: return run_leaf<16, 8, 16>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
    case 32: return run_leaf<32, 8, 16>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
    case 64: return run_leaf<64, 8, 8>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_tslu_node(int W, const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity,
                             int w, int* ids, int* cnt, double* vals, cudaStream_t st, const RootOut* rootp) {
  const RootOut root = rootp ? *rootp : RootOut{};
  switch (W) {
    case 16: return run_node<16, 8, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root);
    case 32: return run_node<32, 8, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root);
    case 64: return run_node<64, 8, 8>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_tslu_panel_factor(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w, int n,
                                     const int* root_ids, const int* root_cnt, double* U, int64_t* piv,
                                     uint8_t* chosen, double* lpanel, unsigned long long* status, cudaStream_t st,
                                     int packed) {
  note_launch(); tslu_panel_factor_kernel<<<1, 512, 0, st>>>(src, lds, rows, row0, p0, w, n, root_ids, root_cnt, U, piv, chosen,
                                              lpanel, status, packed);
  return cudaGetLastError();
}
cudaError_t launch_l11_fixup(double* L11, int n, cudaStream_t st) {
  note_launch(); l11_fixup_kernel<<<n, 128, 0, st>>>(L11, n);
  return cudaGetLastError();
}
cudaError_t launch_gather_rows(const double* src, int64_t lds, const int64_t* ids, int64_t row0, int cnt, int ncols,
                               double* dst, int64_t ldd, cudaStream_t st) {
  note_launch(); gather_rows_kernel<<<cnt, 128, 0, st>>>(src, lds, ids, row0, cnt, ncols, dst, ldd);
  return cudaGetLastError();
}
cudaError_t launch_pivpos(const int64_t* piv, int n, int64_t row0, int64_t rows, int* pivpos, cudaStream_t st) {
  note_launch(); pivpos_kernel<<<ceil_div(n, 128), 128, 0, st>>>(piv, n, row0, rows, pivpos);
  return cudaGetLastError();
}

}  // namespace rlhc
