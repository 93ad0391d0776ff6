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

#ifdef RLHC_TSLU_TRACE
// probe builds only (tools/probe/ptslu.cu): per-block phase timestamps
__device__ unsigned long long g_tslu_trace[4096 * 8];
// distinct trace rows per level of the cfg2 tree (grids of 256, 64, 16, 4, 1 blocks)
__device__ __forceinline__ int tslu_trace_base(int g) {
  return g == 256 ? 0 : g == 64 ? 256 : g == 16 ? 320 : g == 4 ? 336 : g == 1 ? 340 : 0;
}
#define TSLU_TRACE(k)                                                                     \
  if (threadIdx.x == 0) {                                                                 \
    unsigned long long t_;                                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
    g_tslu_trace[(blockIdx.x + tslu_trace_base(gridDim.x)) * 8 + (k)] = t_;               \
  }
#else
#define TSLU_TRACE(k)
#endif

// Candidate staging: the R x w panel block is read row-contiguously (coalesced) into shared
// memory -- the step-column area, free until the select starts -- with row stride W + 1
// (conflict-free column reads), then each warp takes its round-robin columns into registers.
template <int W, int NW, int RS>
RLHC_DEV double* sel_stage(SelSmem<W, NW, RS>& sm) { return &sm.col[0][0]; }
template <int W, int NW, int RS>
RLHC_DEV void sel_fill(const double* stg, double (&a)[RS][W / NW]) {
  const int lane = lane_id(), wp = warp_id();
#pragma unroll
  for (int s = 0; s < RS; s++)
#pragma unroll
    for (int c = 0; c < W / NW; c++) a[s][c] = stg[(s * 32 + lane) * (W + 1) + wp + NW * c];
}
// ov (slot values, row stride W) <- the winners' rows: a warp per row, lanes along columns
template <int W, int NW, typename RowPtr>
RLHC_DEV void write_slot_rows(double* __restrict__ ov, int steps, int w, RowPtr row_of) {
  const int lane = lane_id(), wp = warp_id();
#pragma unroll
  for (int k = 0; k < (W + NW - 1) / NW; k++) {
    const int q = wp + NW * k;
    if (q < steps) {
      const double* src = row_of(q);
#pragma unroll
      for (int c0 = 0; c0 < W; c0 += 32)
        if (c0 + lane < w) ov[q * W + c0 + lane] = src[c0 + lane];
    }
  }
}

// Leaf select: leaf = global row block [leaf*R, leaf*R + R) of the LOCAL rows
// (global id = row0 + local row).  src: current values (X for the first panel, the
// trailing matrix afterwards), panel columns [p0, p0 + w).  Output level slot = leaf.
template <int W, int NW, int RS>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_leaf_kernel(const double* __restrict__ src, int64_t lds, int64_t rows_all, int64_t leaf_rows, int64_t row0, int p0, int w,
                 const uint8_t* __restrict__ chosen, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals, RootOut root, unsigned long long* finite_status) {
  constexpr int R = 32 * RS;
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelSmem<W, NW, RS>& sm = *reinterpret_cast<SelSmem<W, NW, RS>*>(sel_raw);
  TSLU_TRACE(0)
  pdl_trigger();
  sel_init(sm, root.U, root.n);
  const int lane = lane_id();
  const int64_t rb = (int64_t)blockIdx.x * leaf_rows;
  const int64_t rows = rows_all < rb + leaf_rows ? rows_all : rb + leaf_rows;  // end of this leaf
  double* stg = sel_stage(sm);
  // staging: a warp per row, lanes along the columns, every copy in flight at once
  // (cp.async), rows past the end and columns past w zero-filled
#pragma unroll 4
  for (int q = warp_id(); q < R; q += NW) {
    const int64_t r = rb + q;
#pragma unroll
    for (int c0 = 0; c0 < W; c0 += 32) {
      const int c = c0 + lane;
      if (c < W) {
        const bool in = r < rows && c < w;
        cp_async8(stg + q * (W + 1) + c, in ? src + r * lds + p0 + c : src, in ? 8 : 0);
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // single-panel pipelines fold the input check (check_finite_kernel's semantics: the
  // smallest non-finite element index i*n + j wins) into this pass over X
  if (finite_status) {
    for (int idx = threadIdx.x; idx < R * W; idx += blockDim.x) {
      const int q = idx / W, c = idx - q * W;
      if (rb + q < rows && c < w && !isfinite(stg[q * (W + 1) + c]))
        report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, (rb + q) * w + c);
    }
  }
  int gid[RS];
  unsigned act = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int64_t r = rb + s * 32 + lane;
    const bool ok = r < rows && !(chosen && chosen[r]);
    act |= (ok ? 1u : 0u) << s;
    gid[s] = (int)(row0 + r);
  }
  double a[RS][W / NW];
  sel_fill<W, NW, RS>(stg, a);
  TSLU_TRACE(2)
  const int steps = gepp_select<W, NW, RS>(a, act, gid, w, sm);
  TSLU_TRACE(3)
  if (root.U) sel_root_finish(sm, steps, w, root);
  int* oi = out_ids + (size_t)blockIdx.x * W;
  if (threadIdx.x == 0) out_cnt[blockIdx.x] = steps;
  for (int e = threadIdx.x; e < W; e += blockDim.x) oi[e] = e < steps ? sm.out_id[e] : -1;
  if (out_vals)
    write_slot_rows<W, NW>(out_vals + (size_t)blockIdx.x * W * W, steps, w,
                           [&](int q) { return src + (rb + sm.out_src[q]) * lds + p0; });
  TSLU_TRACE(4)
}

// Node select: node = children [node*arity, node*arity + arity) of the level below;
// loaded entry j -> child (j / w), entry (j % w).  The entries are sorted by global id into
// the candidate order (select.cuh's tie rule; slots list their winners in pivot order).
// Values are the stored current panel values of the candidates (not the eliminated ones).
template <int W, int NW, int RS>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_node_kernel(const int* __restrict__ in_ids, const int* __restrict__ in_cnt, const double* __restrict__ in_vals,
                 int nslots_in, int arity, int w, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals, RootOut root, RowSrc rsrc) {
  constexpr int R = 32 * RS;
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelSmem<W, NW, RS>& sm = *reinterpret_cast<SelSmem<W, NW, RS>*>(sel_raw);
  TSLU_TRACE(0)
  pdl_trigger();
  sel_init(sm, root.U, root.n);
  pdl_wait();  // the level below (launched before this one) has completed
  const int lane = lane_id();
  const int c0 = blockIdx.x * arity;
  // entry ids (INT_MAX: no entry) in cgid, which the select first writes after this
  // kernel's last read of them (a barrier apart)
  int* eid = sm.cgid;
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    const int ci = j / w, e = j - ci * w, child = c0 + ci;
    const bool ok = ci < arity && child < nslots_in && e < in_cnt[child];
    eid[j] = ok ? in_ids[child * W + e] : INT_MAX;
    sm.perm[j] = -1;
  }
  __syncthreads();
  // rank of each entry among the valid ones (ids are unique): candidate order = id order
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    const int my = eid[j];
    if (my == INT_MAX) continue;
    int rank = 0;
    const int4* e4 = reinterpret_cast<const int4*>(eid);
#pragma unroll 8
    for (int k4 = 0; k4 < R / 4; k4++) {
      const int4 v = e4[k4];
      rank += (v.x < my) + (v.y < my) + (v.z < my) + (v.w < my);
    }
    sm.perm[rank] = j;
  }
  __syncthreads();
  TSLU_TRACE(1)
  int gid[RS];
  unsigned act = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int j = sm.perm[s * 32 + lane];
    act |= (j >= 0 ? 1u : 0u) << s;
    gid[s] = j >= 0 ? eid[j] : INT_MAX;
  }
  double* stg = sel_stage(sm);
#pragma unroll 4
  for (int q = warp_id(); q < R; q += NW) {
    const int j = sm.perm[q];
    const int ci = j / w, e = j - ci * w;
    const double* row = rsrc.src ? rsrc.src + (j >= 0 ? (int64_t)eid[j] - rsrc.row0 : 0) * rsrc.lds + rsrc.p0
                                 : in_vals + (size_t)((c0 + ci) * W + e) * W;
#pragma unroll
    for (int cc = 0; cc < W; cc += 32) {
      const int c = cc + lane;
      if (c < W) {
        const bool in = j >= 0 && c < w;
        cp_async8(stg + q * (W + 1) + c, in ? row + c : (const double*)in_cnt, in ? 8 : 0);  // 0 bytes: no read
      }
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double a[RS][W / NW];
  sel_fill<W, NW, RS>(stg, a);
  TSLU_TRACE(2)
  const int steps = gepp_select<W, NW, RS>(a, act, gid, w, sm);
  TSLU_TRACE(3)
  if (root.U) sel_root_finish(sm, steps, w, root);
  int* oi = out_ids + (size_t)blockIdx.x * W;
  if (threadIdx.x == 0) out_cnt[blockIdx.x] = steps;
  for (int q = threadIdx.x; q < W; q += blockDim.x) oi[q] = q < steps ? sm.out_id[q] : -1;
  if (out_vals)
    write_slot_rows<W, NW>(out_vals + (size_t)blockIdx.x * W * W, steps, w, [&](int q) {
      if (rsrc.src) return rsrc.src + ((int64_t)sm.out_id[q] - rsrc.row0) * rsrc.lds + rsrc.p0;
      const int j = sm.perm[sm.out_src[q]];
      const int ci = j / w, e = j - ci * w;
      return in_vals + (size_t)((c0 + ci) * W + e) * W;
    });
  TSLU_TRACE(4)
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
static cudaError_t run_leaf(int64_t leaf_rows, const double* src, int64_t lds, int64_t rows, int64_t row0, int p0,
                            int w, const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st,
                            const RootOut& root, unsigned long long* finite_status) {
  if (leaf_rows < 1 || leaf_rows > 32 * RS) return cudaErrorInvalidValue;
  int nleaves = (int)ceil_div<int64_t>(rows, leaf_rows);
  constexpr int smem = (int)sizeof(SelSmem<W, NW, RS>);
  static DevFlags attr_l, attr_n;  // per device and instantiation
  if (cudaError_t e = smem_attr(attr_l, tslu_leaf_kernel<W, NW, RS>, smem)) return e;
  if (cudaError_t e = smem_attr(attr_n, tslu_node_kernel<W, NW, RS>, smem)) return e;
  note_launch(); tslu_leaf_kernel<W, NW, RS><<<nleaves, 32 * NW, smem, st>>>(src, lds, rows, leaf_rows, row0, p0, w, chosen, ids, cnt, vals,
                                                                            root, finite_status);
  return cudaGetLastError();
}
template <int W, int NW, int RS>
static cudaError_t run_node(const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity, int w,
                            int* ids, int* cnt, double* vals, cudaStream_t st, const RootOut& root,
                            const RowSrc& rsrc) {
  int nout = ceil_div(nin, arity);
  constexpr int smem = (int)sizeof(SelSmem<W, NW, RS>);
  static DevFlags attr_l, attr_n;
  if (cudaError_t e = smem_attr(attr_l, tslu_leaf_kernel<W, NW, RS>, smem)) return e;
  if (cudaError_t e = smem_attr(attr_n, tslu_node_kernel<W, NW, RS>, smem)) return e;
  note_launch();
  return launch_pdl(tslu_node_kernel<W, NW, RS>, dim3(nout), dim3(32 * NW), smem, st, in_ids, in_cnt, in_vals, nin,
                    arity, w, ids, cnt, vals, root, rsrc);
}

cudaError_t launch_tslu_leaf(int W, int64_t leaf_rows, const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                             const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st,
                             const RootOut* rootp, unsigned long long* finite_status) {
  const RootOut root = rootp ? *rootp : RootOut{};
  switch (W) {
    case 16: return run_leaf<16, 8, 16>(leaf_rows, src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
    case 32: return run_leaf<32, 8, 16>(leaf_rows, src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
    case 64: return run_leaf<64, 8, 8>(leaf_rows, src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st, root,
                                             finite_status);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_tslu_node(int W, const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity,
                             int w, int* ids, int* cnt, double* vals, cudaStream_t st, const RootOut* rootp,
                             const RowSrc* rowsp) {
  const RootOut root = rootp ? *rootp : RootOut{};
  const RowSrc rsrc = rowsp ? *rowsp : RowSrc{};
  switch (W) {
    case 16: return run_node<16, 8, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root, rsrc);
    case 32: return run_node<32, 8, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root, rsrc);
    case 64: return run_node<64, 8, 8>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st, root, rsrc);
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
