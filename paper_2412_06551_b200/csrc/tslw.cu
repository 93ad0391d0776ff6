// tslw.cu -- warp-level tournament LU "PX = LU" under the
// pivot contract of DESIGN.md R#3-R#5 with 16-column panels, 128-row leaves and nodes of
// up to 8 children: the default contract (rlhc_default_tslu_cfg).
//
// One WARP runs one tournament node: 128 candidate rows x 16 panel columns in registers,
// lane = candidate row (4 slots per lane), so a GEPP step needs no communication beyond
// the warp (three warp reductions for the pivot, the pivot row through 2 KB of per-warp
// shared memory) and many nodes run side by side on every SM.
//
// Panels are LEFT-LOOKING with L kept in the L buffer (the caller's Q buffer in the
// pipelines): for panel j (columns [p0, p0+16)) the leaf kernel
//   1. turns the previous panel's Schur values S_{j-1} (kept in L's columns [p0-16, p0))
//      into L columns by forward substitution with U's diagonal block (in place);
//   2. forms S_j = X[:, p0:p0+w] - L[:, :p0] U[:p0, p0:p0+w] (fma chain in increasing k)
//      and stores it in L's columns [p0, p0+w);
//   3. selects its leaf's 16 winners.
// Node kernels read their candidates' S_j rows by global id.  The root emits piv, U's
// diagonal block, 1/diag(U) and the in-panel multipliers; tslw_urows_kernel completes the
// panel's U rows right of the panel.  After the last panel, tslw_lfinal_kernel converts
// the last S into L and tslw_fixup_kernel gives the pivot rows their L11 rows.
// Every element of S, L and U is the oracle's fma chain (oracle ora_tslu / l_row: the
// elimination and the substitution are the same chain), so piv, U, L11 and L are bit-exact.
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace rlhc {

#ifdef RLHC_TSLW_TRACE
// probe builds only (tools/probe/ptslw.cu): per-warp phase records
__device__ unsigned long long g_tw[1 << 16][8];
__device__ unsigned g_twn;
#define TW_T(v) long long v = clock64(); unsigned long long v##g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v##g));
#define TW_REC(tag, a, b, c, d)                                                              \
  if (lane_id() == 0) {                                                                      \
    unsigned i_ = atomicAdd(&g_twn, 1u);                                                     \
    if (i_ < (1u << 16)) {                                                                   \
      g_tw[i_][0] = tag; g_tw[i_][1] = p0; g_tw[i_][2] = gridDim.x; g_tw[i_][3] = a##g;      \
      g_tw[i_][4] = b - a; g_tw[i_][5] = c - b; g_tw[i_][6] = d - c; g_tw[i_][7] = d##g;     \
    }                                                                                        \
  }
__device__ long long g_stp[64];
// per level of the climbing warp: select start/end, arrival done, node staged (globaltimer ns)
__device__ unsigned long long g_lv[1 << 14][6];
__device__ unsigned g_lvn;
#define TW_G(v) unsigned long long v; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
#define TW_LV(lev, a, b, c, d)                                                              \
  if (lane_id() == 0) {                                                                     \
    unsigned i_ = atomicAdd(&g_lvn, 1u);                                                    \
    if (i_ < (1u << 14)) { g_lv[i_][0] = p0; g_lv[i_][1] = lev; g_lv[i_][2] = a; g_lv[i_][3] = b; g_lv[i_][4] = c; g_lv[i_][5] = d; } \
  }
#define TW_STEP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_stp[i] = clock64();
#else
#define TW_T(v)
#define TW_REC(tag, a, b, c, d)
#define TW_STEP(i)
#define TW_G(v)
#define TW_LV(lev, a, b, c, d)
#endif


constexpr int WW = kTslwPanel;  // panel width
constexpr int RS = 4;           // candidate slots per lane
constexpr int WR = 32 * RS;     // candidate rows per warp (= leaf rows, >= arity * WW)
constexpr int WPB = 4;          // warps (tournament nodes) per CTA

constexpr int TS = 18;          // row stride (doubles) of the staging tile: 16-byte rows, conflict-free LDS.128 by row

struct alignas(16) WSel {
  double tile[WR * TS];  // staging of the node's candidate rows (128 x 16)
  double prow[WW][WW];   // step t: the pivot row (c >= t: U values; c < t: multipliers, root only)
  double r[WW];          // 1 / pivot of step t
  int sid[WR];           // global id of candidate (tile row) c (INT_MAX: none)
  int rank[WR];          // position of candidate c in increasing-id order (the tie-break key)
  int win[WW];           // candidate (tile row) of the winner of step t
  int zero[WW];          // 1: zero pivot column at step t (R#5: no update)
};

// Pivot row of step t (slot ps of the pivot lane), columns [c0, WW) -> dst (c0 even);
// only the pivot lane runs it.
#define TSLW_ROW_CASE(S)                                                                      \
  case S: {                                                                                   \
    _Pragma("unroll") for (int c = 0; c < WW; c += 2) if (c >= c0)                            \
      *reinterpret_cast<double2*>(dst + c) = make_double2(a[S][c], a[S][c + 1]);               \
  } break;
RLHC_DEV void write_prow(const double (&a)[RS][WW], int ps, double* dst, int c0) {
  switch (ps) {
    TSLW_ROW_CASE(0) TSLW_ROW_CASE(1) TSLW_ROW_CASE(2) TSLW_ROW_CASE(3)
    default: break;
  }
}
#undef TSLW_ROW_CASE
// Generic GEPP select of one warp (definition: oracle gepp_select, R#4-R#5):
// any step count, zero pivot columns, reciprocals outside rcp_newton's window.
// a[s][c]: candidate s*32 + lane, panel column c; candidates are in increasing global-id
// order over the active ones (bit s of act), so "ties -> smallest id" is "smallest
// candidate index".  sm.win / sm.prow (whole rows) / sm.r / sm.zero hold the winners.
// The maximum of |a| is taken on the bit patterns (sign cleared) of the 32-bit halves:
// high words, then low words among the rows attaining the high maximum.
RLHC_DEV void wsel_gepp(double (&a)[RS][WW], unsigned act, int steps, const int (&rk)[RS], WSel& sm) {
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < WW; t++) {
    if (t < steps) {
      int hi[RS];
      unsigned lo[RS];
#pragma unroll
      for (int s = 0; s < RS; s++) {
        hi[s] = ((act >> s) & 1u) ? (__double2hiint(a[s][t]) & 0x7fffffff) : -1;
        lo[s] = (unsigned)__double2loint(a[s][t]);
      }
      int mh = max(max(hi[0], hi[1]), max(hi[2], hi[3]));
      mh = __reduce_max_sync(0xffffffffu, mh);
      unsigned ml = 0;
#pragma unroll
      for (int s = 0; s < RS; s++) ml = max(ml, hi[s] == mh ? lo[s] : 0u);
      ml = __reduce_max_sync(0xffffffffu, ml);
      const double pabs = __longlong_as_double((long long)(((unsigned long long)(unsigned)mh << 32) | ml));
      double rabs = rcp_newton(pabs);
      int kr = INT_MAX;  // smallest rank (= smallest id) among this lane's rows attaining the maximum
#pragma unroll
      for (int s = 0; s < RS; s++) kr = (hi[s] == mh && lo[s] == ml) ? min(kr, rk[s]) : kr;
      const int prank = __reduce_min_sync(0xffffffffu, kr);
      const bool zero = (mh | (int)ml) == 0;
      if (!zero && !rcp_newton_ok(mh)) rabs = rcp_slow(pabs);  // warp-uniform, rare
      int ps = -1;
#pragma unroll
      for (int s = 0; s < RS; s++) ps = rk[s] == prank ? s : ps;
      if (ps >= 0) {  // the pivot's lane
        act &= ~(1u << ps);
        write_prow(a, ps, &sm.prow[t][0], 0);
        sm.win[t] = ps * 32 + lane;
        sm.zero[t] = zero ? 1 : 0;
      }
      __syncwarp();
      if (!zero) {
        const double r = sm.prow[t][t] < 0.0 ? -rabs : rabs;  // drcp(-x) == -drcp(x)
        if (lane == 0) sm.r[t] = r;
        double l[RS];
#pragma unroll
        for (int s = 0; s < RS; s++) {
          l[s] = __dmul_rn(a[s][t], r);
          a[s][t] = l[s];
        }
#pragma unroll
        for (int c = t + 1; c < WW; c++) {
          const double u = sm.prow[t][c];
#pragma unroll
          for (int s = 0; s < RS; s++) a[s][c] = __fma_rn(-l[s], u, a[s][c]);
        }
      } else if (lane == 0) {
        sm.r[t] = 0.0;
      }
    }
  }
  __syncwarp();
}

// Fast select: 16 full steps as a compact loop (the code stays hot in the instruction
// cache; a lone warp runs every tournament node on the critical path).  Registers are
// ROTATED: at step t, a[s][k] holds column t + k, so every index is static.  The update
// of step t is split: column t + 1 right away (the next pivot search needs it), the
// other columns at the start of step t + 1, in the shadow of its warp reductions.  The
// pivot's sign rides on the index reduction (key = candidate index * 2 + sign).  Returns
// false if a pivot column was zero or a pivot fell outside rcp_newton's window (the
// caller reruns the generic select).  prow[t][j] = the pivot row's column t + j (rotated).
// pending update of step t - 1 for rotated columns [K0, K1): a[k] = a[k+1] - l u[k+1]
template <int K0, int K1>
RLHC_DEV void wsel_pend(double (&a)[RS][WW], const double (&lp)[RS], const double* up) {
#pragma unroll
  for (int k = K0; k < K1; k++) {
    const double u = up[k + 1];
#pragma unroll
    for (int s = 0; s < RS; s++) a[s][k] = __fma_rn(-lp[s], u, a[s][k + 1]);
  }
}

// One step; PEND: apply step t - 1's pending update (t > 0), in chunks placed after each
// warp reduction so that the DFMAs issue in the reductions' latency shadows.
// KMAX: the pending update writes slots [1, KMAX) only (at step t the live columns are
// t .. 15, i.e. slots 0 .. 15 - t: KMAX = 16 - t is enough, so the rotation narrows).
template <bool PEND, int KMAX = WW - 1>
RLHC_DEV void wsel_step(double (&a)[RS][WW], double (&lp)[RS], unsigned& act, bool& bad, int t, const int (&rk)[RS],
                        WSel& sm) {
  const int lane = lane_id();
  TW_STEP(t)
  const double* up = PEND ? &sm.prow[t - 1][0] : nullptr;
  int hi[RS];
  unsigned lo[RS];
#pragma unroll
  for (int s = 0; s < RS; s++) {
    hi[s] = ((act >> s) & 1u) ? (__double2hiint(a[s][0]) & 0x7fffffff) : -1;
    lo[s] = (unsigned)__double2loint(a[s][0]);
  }
  int mh = max(max(hi[0], hi[1]), max(hi[2], hi[3]));
  mh = __reduce_max_sync(0xffffffffu, mh);
  if (PEND) wsel_pend<1, (KMAX < 6 ? KMAX : 6)>(a, lp, up);
  unsigned ml = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) ml = max(ml, hi[s] == mh ? lo[s] : 0u);
  ml = __reduce_max_sync(0xffffffffu, ml);
  if (PEND) wsel_pend<(KMAX < 6 ? KMAX : 6), (KMAX < 10 ? KMAX : 10)>(a, lp, up);
  const double rabs = rcp_newton(__longlong_as_double((long long)(((unsigned long long)(unsigned)mh << 32) | ml)));
  int key = INT_MAX;
#pragma unroll
  for (int s = RS - 1; s >= 0; s--)
    key = (hi[s] == mh && lo[s] == ml) ? ((rk[s] << 1) | (int)((unsigned)__double2hiint(a[s][0]) >> 31)) : key;
  key = __reduce_min_sync(0xffffffffu, key);
  if (PEND) {
    wsel_pend<(KMAX < 10 ? KMAX : 10), KMAX>(a, lp, up);
    if (KMAX == WW - 1) {
#pragma unroll
      for (int s = 0; s < RS; s++) a[s][WW - 1] = 0.0;
    }
  }
  bad |= (mh | (int)ml) == 0 || !rcp_newton_ok(mh);
  const int prank = key >> 1;
  const double r = (key & 1) ? -rabs : rabs;
  int ps = -1;
#pragma unroll
  for (int s = 0; s < RS; s++) ps = rk[s] == prank ? s : ps;
  if (ps >= 0) {  // the pivot lane publishes its row
    act &= ~(1u << ps);
    write_prow(a, ps, &sm.prow[t][0], 0);
    sm.win[t] = ps * 32 + lane;
  }
  if (lane == 0) {
    sm.r[t] = r;
    sm.zero[t] = 0;
  }
  __syncwarp();
  const double u1 = sm.prow[t][1];
#pragma unroll
  for (int s = 0; s < RS; s++) {
    lp[s] = __dmul_rn(a[s][0], r);
    a[s][0] = __fma_rn(-lp[s], u1, a[s][1]);
  }
}

RLHC_DEV bool wsel_fast(double (&a)[RS][WW], unsigned act, const int (&rk)[RS], WSel& sm) {
  bool bad = false;
  double lp[RS];
  wsel_step<false>(a, lp, act, bad, 0, rk, sm);
  // step 0 left columns 2.. unrotated and un-updated: the pending form of steps >= 1
#pragma unroll 1
  for (int t = 1; t < 4; t++) wsel_step<true, WW - 1>(a, lp, act, bad, t, rk, sm);
#pragma unroll 1
  for (int t = 4; t < 8; t++) wsel_step<true, 12>(a, lp, act, bad, t, rk, sm);
#pragma unroll 1
  for (int t = 8; t < 12; t++) wsel_step<true, 8>(a, lp, act, bad, t, rk, sm);
#pragma unroll 1
  for (int t = 12; t < WW; t++) wsel_step<true, 4>(a, lp, act, bad, t, rk, sm);
  __syncwarp();
  TW_STEP(WW)
  return !bad;
}

// Outputs of a node: ids of the winners in pivot order; at the root also piv, chosen,
// U's diagonal block, 1/diag(U) and rank errors.  rot: prow rows rotated (fast select:
// U(t, t + j) = prow[t][j]); else prow[t][c] = column c.
RLHC_DEV void wsel_emit(const WSel& sm, int steps, int w, int slot, int* out_ids, int* out_cnt, double* out_vals,
                        const TslwRoot& ro, int p0, bool rot) {
  const int lane = lane_id();
  // the slot: every lane writes a part; the climb's __syncwarp orders these writes before
  // lane 0's release (atom.acq_rel.gpu is cumulative), as a CTA barrier before one thread's
  // release publishes the whole CTA's writes
  if (lane == 0) out_cnt[slot] = steps;
  if (lane < WW) out_ids[slot * WW + lane] = lane < steps ? sm.sid[sm.win[lane]] : -1;
  if (out_vals && !ro.U) {  // the winners' (original) panel rows: the parent reads them in one pass
    double2* ov = reinterpret_cast<double2*>(out_vals + (size_t)slot * WW * WW);
#pragma unroll
    for (int j = 0; j < WW * WW / 2 / 32; j++) {
      const int e = j * 32 + lane, q = e / (WW / 2), c = e % (WW / 2);
      if (q < steps) ov[e] = reinterpret_cast<const double2*>(sm.tile + sm.win[q] * TS)[c];
    }
  }
  if (!ro.U) return;
  if (lane == 0 && steps < w) report(ro.status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + steps);
  if (lane < steps) {
    const int gid = sm.sid[sm.win[lane]];
    ro.piv[p0 + lane] = gid;
    ro.chosen[gid - ro.row0] = 1;
    ro.rd[p0 + lane] = sm.r[lane];
    if (sm.zero[lane]) report(ro.status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + lane);
  }
  for (int e = lane; e < WW * WW; e += 32) {
    const int t = e / WW, c = e - t * WW;
    if (t < steps && c < w && c >= t) ro.U[(int64_t)(p0 + t) * ro.n + p0 + c] = rot ? sm.prow[t][c - t] : sm.prow[t][c];
  }
}

// Forward substitution of one row over a 16-column block, RIGHT-looking: l[k] = acc_k *
// rd(k), then acc_c -= l[k] u(k, c) for c > k.  Per element these are the fma chain over k
// in increasing order and the final product of the left-looking loop (the select's own ops),
// but the critical path is 16 steps instead of 120 dependent fmas.  Columns >= lim untouched.
template <typename UF, typename RF>
RLHC_DEV void subst_row_rl(double (&l)[WW], int lim, UF u, RF rd) {
#pragma unroll
  for (int k = 0; k < WW; k++) {
    if (k < lim) {
      l[k] = __dmul_rn(l[k], rd(k));
#pragma unroll
      for (int c = k + 1; c < WW; c++)
        if (c < lim) l[c] = __fma_rn(-l[k], u(k, c), l[c]);
    }
  }
}

// Candidates' rows from the staging tile (row c*TS) -> registers; zero for inactive rows and
// columns >= w.
RLHC_DEV void tile_to_regs(const double* tile, int w, double (&a)[RS][WW]) {
  const int lane = lane_id();
#pragma unroll
  for (int s = 0; s < RS; s++)
#pragma unroll
    for (int c = 0; c < WW; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(tile + (s * 32 + lane) * TS + c);
      a[s][c] = c < w ? v.x : 0.0;
      a[s][c + 1] = c + 1 < w ? v.y : 0.0;
    }
}

// Select on the candidates held in the tile (fast path, else the generic one), then emit.
RLHC_DEV void select_and_emit(WSel& sm, unsigned act, int w, int slot, int* out_ids, int* out_cnt, double* out_vals,
                              const TslwRoot& ro, int p0) {
  double a[RS][WW];
  int rk[RS];
#pragma unroll
  for (int s = 0; s < RS; s++) rk[s] = sm.rank[s * 32 + lane_id()];
  tile_to_regs(sm.tile, w, a);
  const int cnt = __reduce_add_sync(0xffffffffu, __popc(act));
  const int steps = min(cnt, w);
  bool done = false;
  if (steps == WW) done = wsel_fast(a, act, rk, sm);
  if (!done) {
    if (steps == WW) tile_to_regs(sm.tile, w, a);  // the fast attempt modified a
    wsel_gepp(a, act, steps, rk, sm);
  }
  wsel_emit(sm, steps, w, slot, out_ids, out_cnt, out_vals, ro, p0, done);
}

// 16-byte L2 copy (bypasses L1: rows written by other SMs in this kernel); src_bytes < 16
// zero-fills the rest
RLHC_DEV void cp_async16_cg(void* smem_ptr, const void* gptr, int src_bytes) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gptr), "r"(src_bytes));
}
RLHC_DEV int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// The candidates' S_j rows (global id sm.sid[q], columns [p0, p0+w)) -> tile rows q.
// v16: rows 16-byte aligned (even ldl, aligned base): 16-byte L2 copies, 4 rows per
// instruction; else 8-byte L2 loads.
RLHC_DEV void stage_rows(WSel& sm, int w, const double* Lb, int64_t ldl, int64_t row0, int p0, bool v16,
                          bool wait = true) {
  const int lane = lane_id();
  if (v16) {
    const int ch = lane & 7;
    const int nb = w - 2 * ch;  // valid doubles in this 16-byte chunk
    const int bytes = nb >= 2 ? 16 : (nb == 1 ? 8 : 0);
#pragma unroll 8
    for (int i = 0; i < WR / 4; i++) {
      const int q = 4 * i + (lane >> 3);
      const int id = sm.sid[q];
      const bool ok = id != INT_MAX;
      cp_async16_cg(sm.tile + q * TS + 2 * ch, ok ? Lb + ((int64_t)id - row0) * ldl + p0 + 2 * ch : Lb,
                    ok ? bytes : 0);
    }
    cp_async_commit();
    if (!wait) return;
    cp_async_wait_all();
  } else {
    const int c = lane & 15;
#pragma unroll 8
    for (int i = 0; i < WR / 2; i++) {
      const int q = 2 * i + (lane >> 4);
      const int id = sm.sid[q];
      sm.tile[q * TS + c] = (id != INT_MAX && c < w) ? __ldcg(Lb + ((int64_t)id - row0) * ldl + p0 + c) : 0.0;
    }
  }
  __syncwarp();
}

// First panel (p0 = 0): its Schur values are X's panel columns -- the copy into L's columns
// [0, w) with the input check of those columns.  CTA = 128 rows, coalesced staging through
// shared memory both ways (X is never written: its load is issued before the dependency wait).
constexpr int SR = 128;  // rows per CTA
constexpr int ST = 17;   // tile row stride (doubles)
RLHC_DEV void schur_stage(double* tile, const double* base, int64_t ld, int64_t rb, int64_t rows, int col, int w) {
  const int c = threadIdx.x & 15;
#pragma unroll
  for (int j = 0; j < SR / 8; j++) {
    const int q = (threadIdx.x >> 4) + 8 * j;
    const bool in = rb + q < rows && c < w;
    cp_async8(tile + q * ST + c, in ? base + (rb + q) * ld + col + c : base, in ? 8 : 0);
  }
}
__global__ void __launch_bounds__(SR)
tslw_schur0_kernel(const double* __restrict__ X, int64_t ldx, double* __restrict__ Lb, int64_t ldl, int64_t rows,
                   int w, int n, unsigned long long* finite_status) {
  __shared__ double Bx[SR * ST];
  const int64_t rb = (int64_t)blockIdx.x * SR;
  const int tid = threadIdx.x;
  schur_stage(Bx, X, ldx, rb, rows, 0, w);
  cp_async_commit();
  pdl_trigger();
  pdl_wait();  // L may still be read by the previous call's last kernels
  cp_async_wait_all();
  __syncthreads();
  const int64_t r = rb + tid;
  if (finite_status && r < rows) {
#pragma unroll
    for (int c = 0; c < WW; c++)
      if (c < w && !isfinite(Bx[tid * ST + c])) report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, r * n + c);
  }
  const int c = tid & 15;
#pragma unroll
  for (int j = 0; j < SR / 8; j++) {
    const int q = (tid >> 4) + 8 * j;
    if (rb + q < rows && c < w) Lb[(rb + q) * ldl + c] = Bx[q * ST + c];
  }
}

// The same Schur complement on the FP64 tensor cores, for panels with p0 > 0:
// CTA = 128 rows x 16 columns, 8 warps of 16 x 16 (2 x 2 DMMA m8n8k4 fragments);
// acc = X[:, panel]; acc -= L[:, k] U[k, panel] over k = 0 .. kold-1 in 32-wide chunks
// (double-buffered cp.async), then over the previous panel's 16 columns, whose L values
// the CTA's first 128 threads compute first (row substitution of S_{j-1}) and publish
// both to L and to shared memory.  DMMA m8n8k4 is bitwise the fma chain over its 4 k's
// (profiles/r01_probe_fp64_hbm.txt), so every element is the same increasing-k chain.
constexpr int SD_M = 128, SD_K = 32;
struct SchurDSmem {
  double A[2][SD_M][SD_K + 4];
  double B[2][SD_K][WW + 4];
  double Lt[SD_M][WW + 4];   // L_{j-1} of the CTA's rows (A operand of the last chunk)
  double Ut[WW][WW + 4];     // U[kold + k, p0 + c] (B operand of the last chunk)
  double Ublk[WW][WW + 1];   // the previous panel's diagonal block
  double rdp[WW];
};
// Grouped (GROUP panels share one bulk product, run_tslw): the accumulators start from the
// group's partial Schur values B = X - L[:, :P0] U[:P0, group] kept in Lb's columns (Xs = Lb,
// kbeg = P0), and only k = P0 .. p0-1 remain: the same fma chain, continued.
__global__ void __launch_bounds__(256, 2)
tslw_schur_dmma_kernel(const double* __restrict__ X, int64_t ldx, double* __restrict__ Lb, int64_t ldl, int64_t rows,
                       int p0, int w, int n, const double* __restrict__ U, const double* __restrict__ rd,
                       unsigned long long* finite_status, const double* Xs, int64_t ldxs, int kbeg, int pre_only) {
  extern __shared__ __align__(16) unsigned char sd_raw[];
  SchurDSmem& sm = *reinterpret_cast<SchurDSmem*>(sd_raw);
  const int64_t r0 = (int64_t)blockIdx.x * SD_M;
  const int tid = threadIdx.x, lane = lane_id(), wp = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int kold = p0 - WW;
  const bool al = ((ldl & 1) == 0) && ((((uintptr_t)Lb) & 15) == 0) && ((n & 1) == 0) && ((((uintptr_t)U) & 15) == 0);
  // the accumulators' start: X (never written: read before the dependency wait) or, grouped,
  // the partial Schur values the previous kernels left in Lb (read after it)
  double acc[2][2][2];
  auto init = [&]() {
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int b = 0; b < 2; b++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t gr = r0 + wp * 16 + a * 8 + g;
          const int c = b * 8 + 2 * t + h;
          const double v = (gr < rows && c < w) ? Xs[gr * ldxs + p0 + c] : 0.0;
          // (grouped: X's columns were checked by the bulk product's read of them)
          if (finite_status && Xs == X && !isfinite(v))
            report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, gr * n + p0 + c);
          acc[a][b][h] = v;
        }
  };
  if (Xs == X) init();
  pdl_trigger();
  pdl_wait();
  if (Xs != X) init();
  auto load_chunk = [&](int st, int kc) {
    // A: 128 rows x 32 k (16-byte pairs, 8 per thread); B: 32 k x 16 columns (1 pair per thread)
#pragma unroll
    for (int i = 0; i < SD_M * SD_K / 2 / 256; i++) {
      const int idx = tid + 256 * i;
      const int r = idx / (SD_K / 2), c = 2 * (idx % (SD_K / 2));
      const int64_t gr = r0 + r;
      const int k = kc + c;
      double* dst = &sm.A[st][r][c];
      const double* src = Lb + gr * ldl + k;
      const bool rok = gr < rows;
      if (al) {
        cp_async16_cg(dst, rok && k < kold ? src : Lb, rok && k < kold ? 16 : 0);
      } else {
        cp_async8(dst, (rok && k < kold) ? src : Lb, (rok && k < kold) ? 8 : 0);
        cp_async8(dst + 1, (rok && k + 1 < kold) ? src + 1 : Lb, (rok && k + 1 < kold) ? 8 : 0);
      }
    }
    {
      const int r = tid / (WW / 2), c = 2 * (tid % (WW / 2));
      const int k = kc + r;
      double* dst = &sm.B[st][r][c];
      const double* src = U + (int64_t)k * n + p0 + c;
      if (al) {
        const int nb = (k < kold) ? (c + 1 < w ? 16 : (c < w ? 8 : 0)) : 0;
        cp_async16_cg(dst, nb ? src : U, nb);
      } else {
        cp_async8(dst, (k < kold && c < w) ? src : U, (k < kold && c < w) ? 8 : 0);
        cp_async8(dst + 1, (k < kold && c + 1 < w) ? src + 1 : U, (k < kold && c + 1 < w) ? 8 : 0);
      }
    }
    cp_async_commit();
  };
  // S_{j-1} of the CTA's rows -> Lt (coalesced, 16 threads per row), then the first L chunk
  if (!pre_only) {
    const int c = tid & 15;
#pragma unroll
    for (int j = 0; j < SD_M / 16; j++) {
      const int q = (tid >> 4) + 16 * j;
      const bool in = r0 + q < rows;
      cp_async8(&sm.Lt[q][c], in ? Lb + (r0 + q) * ldl + kold + c : Lb, in ? 8 : 0);
    }
    cp_async_commit();
  }
  if (kold > kbeg) load_chunk(0, kbeg);
  // the previous panel's block, 1/diag, and U[kold.., panel] (pre_only: not needed -- and still
  // being produced by the previous panel's tournament)
  for (int e = tid; e < (pre_only ? 0 : WW * WW); e += 256) {
    const int k = e / WW, c = e - k * WW;
    sm.Ublk[k][c] = U[(int64_t)(kold + k) * n + kold + c];
    sm.Ut[k][c] = c < w ? U[(int64_t)(kold + k) * n + p0 + c] : 0.0;
  }
  if (tid < WW && !pre_only) sm.rdp[tid] = rd ? rd[kold + tid] : __ddiv_rn(1.0, U[(int64_t)(kold + tid) * (n + 1)]);
  if (kold > kbeg && !pre_only) cp_async_wait_1();  // S_{j-1} landed (the L chunk may be in flight)
  else cp_async_wait_all();
  __syncthreads();
  if (tid < SD_M && !pre_only) {  // L_{j-1} of row tid: S_{j-1} -> forward substitution (the select's chain)
    double l[WW];
#pragma unroll
    for (int c = 0; c < WW; c++) l[c] = sm.Lt[tid][c];
    subst_row_rl(l, WW, [&](int k, int c) { return sm.Ublk[k][c]; }, [&](int k) { return sm.rdp[k]; });
#pragma unroll
    for (int c = 0; c < WW; c++) sm.Lt[tid][c] = l[c];
  }
  int st = 0;
  for (int kc = kbeg; kc < kold; kc += SD_K) {
    if (kc + SD_K < kold) {
      load_chunk(st ^ 1, kc + SD_K);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll
    for (int k0 = 0; k0 < SD_K; k0 += 4) {
      double af[2], bf[2];
#pragma unroll
      for (int a = 0; a < 2; a++) af[a] = -sm.A[st][wp * 16 + a * 8 + g][k0 + t];
#pragma unroll
      for (int b = 0; b < 2; b++) bf[b] = sm.B[st][k0 + t][b * 8 + g];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
    st ^= 1;
  }
  __syncthreads();  // Lt complete
  if (!pre_only) {  // L_{j-1} to L (coalesced)
    const int c = tid & 15;
#pragma unroll
    for (int j = 0; j < SD_M / 16; j++) {
      const int q = (tid >> 4) + 16 * j;
      if (r0 + q < rows) Lb[(r0 + q) * ldl + kold + c] = sm.Lt[q][c];
    }
  }
#pragma unroll
  for (int k0 = 0; k0 < (pre_only ? 0 : WW); k0 += 4) {
    double af[2], bf[2];
#pragma unroll
    for (int a = 0; a < 2; a++) af[a] = -sm.Lt[wp * 16 + a * 8 + g][k0 + t];
#pragma unroll
    for (int b = 0; b < 2; b++) bf[b] = sm.Ut[k0 + t][b * 8 + g];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
  // S_j through shared memory (the first A buffer is free), stored coalesced
  double* So = &sm.A[0][0][0];  // [SD_M][SD_K + 4]
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      const int rr = wp * 16 + a * 8 + g, c = b * 8 + 2 * t;
      So[rr * (SD_K + 4) + c] = acc[a][b][0];
      So[rr * (SD_K + 4) + c + 1] = acc[a][b][1];
    }
  __syncthreads();
  {
    const int c = tid & 15;
#pragma unroll
    for (int j = 0; j < SD_M / 16; j++) {
      const int q = (tid >> 4) + 16 * j;
      if (r0 + q < rows && c < w) Lb[(r0 + q) * ldl + p0 + c] = So[q * (SD_K + 4) + c];
    }
  }
}

// The same Schur complement as a warp-specialised TMA pipeline (the default when L is
// TMA-describable): persistent CTAs, one per SM, 128-row tiles; one elected producer thread
// streams, per tile, X's panel columns, S_{j-1} (L's columns [kold, p0)) and then L's columns
// [16 c, 16 c + 16) for c < kold/16 as 128 x 16 boxes (128-byte swizzle) into ST_S stages
// completing on mbarriers; the 8 consumer warps never load A themselves.  Half of them (by
// tile parity) turn S_{j-1} into L_{j-1} (row substitution, thread = row) into a
// double-buffered swizzled Lt and L while the producer keeps streaming the tile's chunks; the
// last k-chunk multiplies Lt after one named barrier.  U[:p0, panel] (B) is staged once per
// CTA.  Same chain per element as tslw_schur_dmma_kernel: acc = X, then k = 0 .. p0-1 in
// increasing order.  (That kernel's two-stage cp.async loop kept the L stream at 49 % of
// HBM: one 32 KB chunk in flight while the last was computed.)
//
// Leaves (ids0 non-null): a tile's 128 rows are one tournament leaf, so the tile's S_j goes
// from the accumulators straight into the staging tile of one of three SELECT warps (tiles
// rotate), which run the tree kernel's own leaf code (select_and_emit: same winners, same
// slot contents) while the consumers stream the next tiles; tslw_tree_kernel then starts at
// level 1.  Saves the tree's re-read of S_j and its leaf wave (a latency chain at 8 warps per
// SM: 25 of the 106 ms LU at cfg5).  Register split by setmaxnreg: the consumer warpgroups
// drop to 128 registers, the producer / select warpgroup rises to 248 (the select holds a
// 128 x 16 tile in registers).  (A first version selected inside the consumer warps, thread
// = row, with named barriers per step: the select lag stalled the stage ring, LU 90 -> 137 ms.)
#ifdef RLHC_ST_PROF  // in-kernel phase clocks of CTA 0 (consumer warp 0, select warp 0), printed per launch
#define STP_DECL long long stp_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, stp_t = clock64(), stp_n = 0;
#define STP(i) { const long long c_ = clock64(); stp_[i] += c_ - stp_t; stp_t = c_; }
#else
#define STP_DECL
#define STP(i)
#endif
constexpr int ST_M = 128, ST_CW = 8;
constexpr int ST_THREADS = 32 * (ST_CW + 4);  // + producer warp, 3 select warps
constexpr int ST_SEL = 3;                     // select warps
// CW consumer warps (8, or 4 in the LIGHT layout: panels whose Schur work is a few chunks are
// bound by the leaf selects, so half the consumers' registers go to NSEL = 6 select warps).
template <int S, int NSEL>
struct __align__(1024) SchurTSmem {
  double A[S][ST_M][WW];     // k chunks (and S_{j-1}), swizzled
  double Lt[2][ST_M][WW];    // L_{j-1} of the tile, swizzled, by tile parity
  double Ublk[WW][WW + 1];
  double rdp[WW];
  unsigned long long full[S], empty[S];
  unsigned long long ready[NSEL], freeb[NSEL];  // select warp k's staging tile: filled / free
  // followed by Bs (U[:p0, panel] in DMMA fragment order: [p0/4][2][32]), in PAIR mode Bs2
  // (U[:p0, next panel]), then (leaves) WSel[NSEL]; only U's rows [16 kbeg, p0) are staged
};
__device__ __forceinline__ int st_off(int row, int k) { return row * WW + ((((k >> 1) ^ row) & 7) << 1) + (k & 1); }
__host__ __device__ inline size_t schur_bs_bytes(int p0) { return (size_t)p0 * WW * sizeof(double); }
template <int S, int NSEL = ST_SEL>
size_t schur_tma_smem_t(int brows, bool pair, bool leaves) {  // brows: rows of U staged (p0 - 16 kbeg)
  return sizeof(SchurTSmem<S, NSEL>) + (pair ? 2 : 1) * schur_bs_bytes(brows) + (leaves ? NSEL * sizeof(WSel) : 0) + 1024;
}
constexpr int ST_LCW = 4, ST_LSEL = 6, ST_LS = 3;  // the LIGHT layout: consumer warps, select warps, stages

// PAIR: the kernel of an even panel j also accumulates, from the same L chunks, the partial
// Schur complement P_{j+1} = X[:, next panel] - L[:, :p0] U[:p0, next panel] of the next panel
// (w2 columns, into L's columns [p0 + 16, p0 + 32)); the odd panel j+1 then starts from P_{j+1}
// (its "X" map over L) and streams no L chunk from HBM (kbeg = nk): every L column is re-read
// once per PAIR of panels.  Same fma chain per element (k increasing), so the same bits.
// PIC (producer in a consumer): lane 0 of consumer warp 0 issues the TMA loads itself -- after it
// releases item q it loads item q + S - 1 (whose stage every consumer released one item ago) --
// and the warp freed carries a FOURTH select warp (the select-bound panels: early and odd ones).
template <int S, bool PAIR, int CW = ST_CW, int NSEL = ST_SEL, bool PIC = false>
__global__ void __launch_bounds__(ST_THREADS, 1)
tslw_schur_tma_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmX,
                      double* __restrict__ Lb, int64_t ldl, int64_t rows, int p0, int w, int n,
                      const double* __restrict__ U, const double* __restrict__ rd, unsigned long long* finite_status,
                      const uint8_t* __restrict__ chosen, int* __restrict__ ids0, int* __restrict__ cnt0,
                      double* __restrict__ vals0, int64_t row0, int kbeg, int w2, int b2) {
  extern __shared__ __align__(1024) unsigned char stm_raw[];
  static_assert(CW == 8 || (CW == 4 && !PAIR), "consumer layouts");
  static_assert(CW + (PIC ? 0 : 1) + NSEL <= ST_THREADS / 32, "warp roles");
  constexpr int H = 8 / CW;  // 64-row halves of the tile per consumer warp
  using Smem = SchurTSmem<S, NSEL>;
  Smem& sm = *reinterpret_cast<Smem*>(stm_raw + ((1024u - (smem_u32(stm_raw) & 1023u)) & 1023u));
  const int bs0 = kbeg * WW;  // U's rows [bs0, p0) are staged (chunks before kbeg are not streamed)
  double* Bs = reinterpret_cast<double*>(&sm + 1);
  double* Bs2 = Bs + (size_t)(p0 - bs0) * WW;  // (PAIR)
  WSel* wsel = reinterpret_cast<WSel*>(reinterpret_cast<unsigned char*>(Bs) + (PAIR ? 2 : 1) * schur_bs_bytes(p0 - bs0));
  const bool leaves = ids0 != nullptr;
  const int tid = threadIdx.x, lane = lane_id(), wp = warp_id();
  const int kold = p0 - WW, nk = kold / WW;
  const int64_t ntiles = ceil_div<int64_t>(rows, ST_M);
  if (tid < S) {
    mbar_init(&sm.full[tid], 1);
    mbar_init(&sm.empty[tid], CW);
  }
  if (tid < NSEL) {
    mbar_init(&sm.ready[tid], CW);
    mbar_init(&sm.freeb[tid], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  // the item stream (both sides walk it in the same order): per tile X's panel columns, (PAIR)
  // the next panel's X columns, S_{j-1}, then L's k chunks kbeg .. nk-1
  struct Prod {
    uint32_t q;
    int64_t tl;
    int c;
    bool done;
  };
  const int pfirst = PAIR ? -3 : -2, pend = p0 ? nk : -1;
  auto prod_issue = [&](Prod& ps) {  // loads the next item (after its stage is free); false: none left
    if (ps.done) return false;
    const int s = (int)(ps.q % S), c = ps.c;
    if (ps.q >= S) mbar_wait(&sm.empty[s], ((ps.q / S) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&sm.full[s])),
                 "r"((uint32_t)(ST_M * WW * 8))
                 : "memory");
    const bool xs = PAIR ? c <= -2 : c == -2;
    const int xc = PAIR ? (c == -3 ? p0 : c == -2 ? p0 + WW : c < 0 ? kold : c * WW)
                        : (c == -2 ? p0 : c < 0 ? kold : c * WW);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(&sm.A[s][0][0])),
        "l"(reinterpret_cast<uint64_t>(xs ? &tmX : &tmL)), "r"(xc), "r"((int)(ps.tl * ST_M)), "r"(smem_u32(&sm.full[s]))
        : "memory");
    ps.q++;
    ps.c++;
    if (ps.c >= 0 && ps.c < kbeg) ps.c = kbeg;
    if (ps.c >= pend) {
      ps.c = pfirst;
      ps.tl += gridDim.x;
      ps.done = ps.tl >= ntiles;
    }
    return true;
  };
  if (wp >= CW) {
    if (CW == 8)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 248;\n" ::: "memory");
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    if (!PIC && wp == CW) {
      // ---------------- producer warp (one lane)
      if (lane != 0) return;
      Prod ps{0u, (int64_t)blockIdx.x, pfirst, (int64_t)blockIdx.x >= ntiles};
      while (prod_issue(ps)) {
      }
      return;
    }
    const int k = wp - CW - (PIC ? 0 : 1);
    if (!leaves || k >= NSEL) return;
    // ---------------- select warp k: the leaves of this CTA's tiles i = k, k + NSEL, ...
    WSel& ws = wsel[k];
    uint32_t i = 0;
    // active rows of tile tl (bit s: row s * 32 + lane); the next tile's flags are loaded before
    // this tile's select so that their latency is off the select chain
    // (volatile loads: issued here, before the select; their values are combined after it)
    auto flags = [&](int64_t tl, unsigned (&f)[RS]) {
#pragma unroll
      for (int s = 0; s < RS; s++) {
        const int64_t r = tl * ST_M + s * 32 + lane;
        f[s] = r < rows ? 0u : 1u;
        if (chosen && r < rows) asm volatile("ld.global.nc.u8 %0, [%1];\n" : "=r"(f[s]) : "l"(chosen + r));
      }
    };
    auto active = [&](const unsigned (&f)[RS]) {
      unsigned act = 0;
#pragma unroll
      for (int s = 0; s < RS; s++) act |= (f[s] ? 0u : 1u) << s;
      return act;
    };
    const int64_t tstep = (int64_t)NSEL * gridDim.x;
    int64_t tl = blockIdx.x + (int64_t)k * gridDim.x;
    unsigned fl[RS] = {1u, 1u, 1u, 1u};
    if (tl < ntiles) flags(tl, fl);
    unsigned act = active(fl);
    STP_DECL
    for (; tl < ntiles; tl += tstep, i++) {
      const int64_t rb = tl * ST_M;
      if (tl + tstep < ntiles) flags(tl + tstep, fl);
#pragma unroll
      for (int s = 0; s < RS; s++) {
        const int64_t r = rb + s * 32 + lane;
        ws.sid[s * 32 + lane] = r < rows ? (int)(row0 + r) : INT_MAX;
        ws.rank[s * 32 + lane] = s * 32 + lane;  // the leaf's rows are in increasing-id order
      }
      STP(0)
      mbar_wait(&sm.ready[k], i & 1);  // the consumers staged S_j of tile tl
      __syncwarp();
      STP(1)
      select_and_emit(ws, act, w, (int)tl, ids0, cnt0, vals0, TslwRoot{}, p0);
      __syncwarp();
      STP(2)
      if (lane == 0) mbar_arrive(&sm.freeb[k]);
      act = active(fl);
#ifdef RLHC_ST_PROF
      stp_n++;
#endif
    }
#ifdef RLHC_ST_PROF
    if (blockIdx.x == 0 && k == 0 && lane == 0)
      printf("STP sel p0=%d CW=%d NSEL=%d tiles=%lld prep=%lld wait_ready=%lld select=%lld\n", p0, CW, NSEL, stp_n,
             stp_[0] / stp_n, stp_[1] / stp_n, stp_[2] / stp_n);
#endif
    return;
  }
  if (CW == 8)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 128;\n" ::: "memory");
  else
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
  // ---------------- consumers (32 CW threads): B in fragment order, the previous panel's block, 1/diag
  for (int e = tid; e < (p0 - bs0) * WW; e += 32 * CW) {
    const int kq = e >> 6, b = (e >> 5) & 1, ln = e & 31;
    const int kk = bs0 + 4 * kq + (ln & 3), c = 8 * b + (ln >> 2);
    Bs[e] = c < w ? U[(int64_t)kk * n + p0 + c] : 0.0;
    if (PAIR) Bs2[e] = c < w2 ? U[(int64_t)kk * n + p0 + WW + c] : 0.0;
  }
  for (int e = tid; e < (p0 ? WW * WW : 0); e += 32 * CW) {
    const int kk = e / WW, c = e - kk * WW;
    sm.Ublk[kk][c] = U[(int64_t)(kold + kk) * n + kold + c];
  }
  if (tid < WW && p0) sm.rdp[tid] = rd ? rd[kold + tid] : __ddiv_rn(1.0, U[(int64_t)(kold + tid) * (n + 1)]);
  asm volatile("bar.sync 1, %0;\n" ::"n"(32 * CW) : "memory");
  const int g = lane >> 2, tq = lane & 3;
  // fragment row a (0, 1) of 64-row half h: conflict-free against the swizzle
  auto frow = [&](int a) { return (a >> 1) * 64 + wp * 16 + 2 * g + (a & 1); };
  constexpr int NA = 2 * H;  // fragment rows per lane
  const bool st16 = (ldl & 1) == 0;                          // (TMA-describable L: base 16-byte aligned)
  uint32_t q = 0, ti = 0;
  int par = 0;
  Prod ps{0u, (int64_t)blockIdx.x, pfirst, (int64_t)blockIdx.x >= ntiles};  // (PIC, warp 0 lane 0)
  // PIC: item qc released by this warp -> load the items up to qc + S - 1
  auto released = [&](uint32_t qc) {
    if (PIC && wp == 0 && lane == 0) {
      while (ps.q < qc + S && prod_issue(ps)) {
      }
    }
  };
  if (PIC && wp == 0 && lane == 0) {
    while (ps.q < (uint32_t)S && prod_issue(ps)) {
    }
  }
  STP_DECL
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x, par ^= 1, ti++) {
    const int64_t r0 = tl * ST_M;
    STP(0)
    double acc[NA][2][2], acc2[1][NA][2][2];  // acc2: PAIR only
    // X's panel columns (zero outside the matrix), with the input check; PAIR: the next panel's
    auto take_x = [&](double (&ac)[NA][2][2], int col0) {
      const int s = (int)(q % S);
      mbar_wait(&sm.full[s], (q / S) & 1);
      const double* xs = &sm.A[s][0][0];
#pragma unroll
      for (int a = 0; a < NA; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const int c = b * 8 + 2 * tq;
          const double2 v = *reinterpret_cast<const double2*>(xs + st_off(frow(a), c));
          ac[a][b][0] = v.x, ac[a][b][1] = v.y;
          if (finite_status) {
            const int64_t gr = r0 + frow(a);
            if (!isfinite(v.x)) report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, gr * n + col0 + c);
            if (!isfinite(v.y)) report(finite_status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, gr * n + col0 + c + 1);
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      released(q);
      q++;
    };
    take_x(acc, p0);
    if (PAIR) take_x(acc2[0], p0 + WW);
    STP(1)
    if (p0) {  // S_{j-1} -> L_{j-1}: thread = tile row, warps 0-3 on even tiles, 4-7 on odd ones
      const int s = (int)(q % S);
      mbar_wait(&sm.full[s], (q / S) & 1);
      STP(2)
      if (CW == 4 || (wp >> 2) == par) {
        const int row = tid & (ST_M - 1);
        const double* src = &sm.A[s][0][0];
        double l[WW];
#pragma unroll
        for (int c = 0; c < WW; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(src + st_off(row, c));
          l[c] = v.x, l[c + 1] = v.y;
        }
        subst_row_rl(l, WW, [&](int kk, int c) { return sm.Ublk[kk][c]; }, [&](int kk) { return sm.rdp[kk]; });
        double* lt = &sm.Lt[par][0][0];
#pragma unroll
        for (int c = 0; c < WW; c += 2) *reinterpret_cast<double2*>(lt + st_off(row, c)) = make_double2(l[c], l[c + 1]);
        if (r0 + row < rows) {
          double* dst = Lb + (r0 + row) * ldl + kold;
          if (st16) {
#pragma unroll
            for (int c = 0; c < WW; c += 2) *reinterpret_cast<double2*>(dst + c) = make_double2(l[c], l[c + 1]);
          } else {
#pragma unroll
            for (int c = 0; c < WW; c++) dst[c] = l[c];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      released(q);
      q++;
      STP(3)
    }
    // two: (PAIR) the chunk also feeds the next panel's partial (chunks c < b2 only)
    auto mma16 = [&](const double* As, int kb, auto two) {  // 16 k's: A stage (swizzled), B rows kb ..
#pragma unroll
      for (int k0 = 0; k0 < WW; k0 += 4) {
        double af[NA], bf[2];
#pragma unroll
        for (int a = 0; a < NA; a++) af[a] = -As[st_off(frow(a), k0 + tq)];
        const double* bp = Bs + (size_t)((kb - bs0 + k0) >> 2) * 64 + lane;
#pragma unroll
        for (int b = 0; b < 2; b++) bf[b] = bp[b * 32];
#pragma unroll
        for (int a = 0; a < NA; a++)
#pragma unroll
          for (int b = 0; b < 2; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        if (PAIR && decltype(two)::value) {
          const double* bp2 = Bs2 + (size_t)((kb - bs0 + k0) >> 2) * 64 + lane;
#pragma unroll
          for (int b = 0; b < 2; b++) bf[b] = bp2[b * 32];
#pragma unroll
          for (int a = 0; a < NA; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) dmma(acc2[0][a][b][0], acc2[0][a][b][1], af[a], bf[b]);
        }
      }
    };
    for (int c = kbeg; c < nk; c++, q++) {
      const int s = (int)(q % S);
      mbar_wait(&sm.full[s], (q / S) & 1);
      if (PAIR && c < b2)
        mma16(&sm.A[s][0][0], c * WW, std::true_type{});
      else
        mma16(&sm.A[s][0][0], c * WW, std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      released(q);
    }
    STP(4)
    if (p0) {
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * CW) : "memory");  // Lt[par] complete
      STP(5)
      if (PAIR && nk < b2)
        mma16(&sm.Lt[par][0][0], kold, std::true_type{});
      else
        mma16(&sm.Lt[par][0][0], kold, std::false_type{});
    }
    auto store = [&](const double (&ac)[NA][2][2], int col0, int wc) {
#pragma unroll
      for (int a = 0; a < NA; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const int64_t gr = r0 + frow(a);
          const int c = b * 8 + 2 * tq;
          if (gr < rows) {
            double* dst = Lb + gr * ldl + col0 + c;
            if (st16 && c + 1 < wc) {
              *reinterpret_cast<double2*>(dst) = make_double2(ac[a][b][0], ac[a][b][1]);
            } else {
              if (c < wc) dst[0] = ac[a][b][0];
              if (c + 1 < wc) dst[1] = ac[a][b][1];
            }
          }
        }
    };
    STP(6)
    store(acc, p0, w);
    if (PAIR) store(acc2[0], p0 + WW, w2);
    STP(7)
    if (leaves) {  // S_j -> the staging tile of select warp ti % ST_SEL (zero outside the panel)
      const int k = (int)(ti % NSEL);
      if (ti >= NSEL) mbar_wait(&sm.freeb[k], ((ti / NSEL) - 1) & 1);
      STP(8)
      double* tile = wsel[k].tile;
#pragma unroll
      for (int a = 0; a < NA; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const int c = b * 8 + 2 * tq;
          *reinterpret_cast<double2*>(tile + frow(a) * TS + c) =
              make_double2(c < w ? acc[a][b][0] : 0.0, c + 1 < w ? acc[a][b][1] : 0.0);
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.ready[k]);
      STP(9)
    }
#ifdef RLHC_ST_PROF
    stp_n++;
#endif
  }
#ifdef RLHC_ST_PROF
  if (blockIdx.x == 0 && tid == 0)
    printf("STP con p0=%d CW=%d NSEL=%d tiles=%lld loop=%lld wait_x=%lld wait_s=%lld subst=%lld chunks=%lld bar=%lld lt_mma=%lld "
           "store=%lld wait_free=%lld stage=%lld\n", p0, CW, NSEL, stp_n, stp_[0] / stp_n, stp_[1] / stp_n, stp_[2] / stp_n,
           stp_[3] / stp_n, stp_[4] / stp_n, stp_[5] / stp_n, stp_[6] / stp_n, stp_[7] / stp_n, stp_[8] / stp_n,
           stp_[9] / stp_n);
#endif
}

// launch the TMA Schur kernel if L is TMA-describable and its shared memory fits; *done
// tells the caller whether it ran, *leaves_done whether it also selected the leaves (ids0
// non-null asks for it: more than one leaf, and room for the leaf buffers).
// mode 0: the panel from X, every L chunk; mode 1 (PAIR): also the next panel's partial Schur
// complement (w2 columns) into L; mode 2: the panel from the partial in L (the odd panel after
// a PAIR), no L chunk from HBM.
static cudaError_t launch_schur_tma(const double* X, int64_t ldx, double* Lb, int64_t ldl, int64_t rows, int p0,
                                    int w, int n, const double* U, const double* rd, unsigned long long* status,
                                    const uint8_t* chosen, int* ids0, int* cnt0, double* vals0, int64_t row0,
                                    cudaStream_t st, bool* done, bool* leaves_done, int mode = 0, int w2 = 0,
                                    int split = -1) {
  *done = false;
  *leaves_done = false;
  static const bool on = [] { const char* e = getenv("RLHC_SCHUR_TMA"); return !e || atoi(e) != 0; }();
  static const bool leaves_on = [] { const char* e = getenv("RLHC_SCHUR_LEAVES"); return !e || atoi(e) != 0; }();
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  const bool pair = mode == 1;
  // split (modes 1 and 2): the partial covers L chunks [0, split) only (-1: all of [0, p0/16)
  // in mode 1, i.e. the odd panel streams no chunk); the odd panel streams [split, p0/16 - 1)
  const int kbeg = mode == 2 ? (split >= 0 ? split : std::max(0, (p0 - WW) / WW)) : 0;
  const int b2 = mode == 1 && split >= 0 ? split : p0 / WW;
  const int brows = p0 - kbeg * WW;
  // LIGHT layout (4 consumer warps, 6 select warps), RLHC_SCHUR_LIGHT=<max p0>: the early panels
  // (p0 <= light_p0) and the odd panels of pairs (no L chunk streamed)
  static const int light_p0 = [] { const char* e = getenv("RLHC_SCHUR_LIGHT"); return e ? atoi(e) : -1; }();
  // P4 layout (the producer inside consumer warp 0, 4 select warps), RLHC_SCHUR_P4=<max p0>: the plain
  // panels up to that p0 and the odd panels of pairs.  Both layouts are measurement knobs, off by
  // default: neither beat the default layout.
  static const int p4_p0 = [] { const char* e = getenv("RLHC_SCHUR_P4"); return e ? atoi(e) : -1; }();
  const bool light_want = leaves_on && ids0 && rows > ST_M && light_p0 >= 0 &&
                          ((mode == 0 && p0 <= light_p0) || (mode == 2 && split < 0)) &&
                          schur_tma_smem_t<ST_LS, ST_LSEL>(brows, false, true) <= 227 * 1024;
  auto smem_of = [&](bool lv) {
    return pair ? schur_tma_smem_t<4>(brows, true, lv) : schur_tma_smem_t<5>(brows, false, lv);
  };
  const bool p4_want = !light_want && leaves_on && ids0 && rows > ST_M && !pair && p4_p0 >= 0 && (p0 <= p4_p0 || mode == 2) &&
                       schur_tma_smem_t<5, 4>(brows, false, true) <= 227 * 1024;
  bool leaves = light_want || p4_want || (leaves_on && ids0 && rows > ST_M && smem_of(true) <= 227 * 1024);
  const size_t smem = light_want ? schur_tma_smem_t<ST_LS, ST_LSEL>(brows, false, true)
                      : p4_want  ? schur_tma_smem_t<5, 4>(brows, false, true)
                                 : smem_of(leaves);
  if (!on || !enc || (ldl & 1) || (ldx & 1) || (reinterpret_cast<uintptr_t>(Lb) & 15) ||
      (reinterpret_cast<uintptr_t>(X) & 15) || smem > 227 * 1024 || rows >= (int64_t(1) << 31))
    return cudaSuccess;
  auto make = [&](CUtensorMap* m, const double* base, int64_t ld, int cols) {
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {WW, ST_M};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  CUtensorMap mL, mX;
  const bool xok = mode == 2 ? make(&mX, Lb, ldl, p0 + w) : make(&mX, X, ldx, pair ? p0 + WW + w2 : p0 + w);
  if (!xok || !make(&mL, p0 ? Lb : X, p0 ? ldl : ldx, p0 ? p0 : w)) return cudaSuccess;
  int dev = 0, sms = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, ST_M), sms));
  note_launch();
  *done = true;
  *leaves_done = leaves;
  if (pair) {
    static DevFlags attr;
    if (cudaError_t e = smem_attr(attr, tslw_schur_tma_kernel<4, true>, 227 * 1024)) return e;
    return launch_pdl(tslw_schur_tma_kernel<4, true>, dim3((unsigned)grid), dim3(ST_THREADS), smem, st, mL, mX, Lb,
                      ldl, rows, p0, w, n, U, rd, status, chosen, leaves ? ids0 : (int*)nullptr, cnt0, vals0, row0,
                      kbeg, w2, b2);
  }
  if (light_want) {
    static DevFlags attr;
    auto kern = tslw_schur_tma_kernel<ST_LS, false, ST_LCW, ST_LSEL>;
    if (cudaError_t e = smem_attr(attr, kern, 227 * 1024)) return e;
    return launch_pdl(kern, dim3((unsigned)grid), dim3(ST_THREADS), smem, st, mL, mX, Lb, ldl, rows, p0, w, n, U, rd,
                      mode == 2 ? (unsigned long long*)nullptr : status, chosen, ids0, cnt0, vals0, row0, kbeg, 0, 0);
  }
  if (p4_want) {
    static DevFlags attr;
    auto kern = tslw_schur_tma_kernel<5, false, ST_CW, 4, true>;
    if (cudaError_t e = smem_attr(attr, kern, 227 * 1024)) return e;
    return launch_pdl(kern, dim3((unsigned)grid), dim3(ST_THREADS), smem, st, mL, mX, Lb, ldl, rows, p0, w, n, U, rd,
                      mode == 2 ? (unsigned long long*)nullptr : status, chosen, ids0, cnt0, vals0, row0, kbeg, 0, 0);
  }
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, tslw_schur_tma_kernel<5, false>, 227 * 1024)) return e;
  return launch_pdl(tslw_schur_tma_kernel<5, false>, dim3((unsigned)grid), dim3(ST_THREADS), smem, st, mL, mX, Lb,
                    ldl, rows, p0, w, n, U, rd, mode == 2 ? (unsigned long long*)nullptr : status, chosen,
                    leaves ? ids0 : (int*)nullptr, cnt0, vals0, row0, kbeg, 0, 0);
}

// The tournament's climb for one warp: select the node held in sm (active mask act) and emit
// it into `slot` of level lev, then, if this warp's child is the last of its parent to arrive,
// run the parent -- up to the root (or level stop_lev).  skip_first: the level-0 slots are
// already emitted (the Schur kernel selected the leaves): start as `slot`'s parent's runner.
RLHC_DEV void tree_climb(WSel& sm, int nleaves, int slot, unsigned act, const int* cids, const double* cvals,
                         int* ids0, int* cnt0, double* vals0, int* idsN, int* cntN, double* valsN, int* arrive,
                         int arity, int stop_lev, const TslwRoot& ro, int p0, int w, bool skip_first) {
  const int lane = lane_id();
  int nsl = nleaves;
  int *oids = ids0, *ocnt = cnt0;
  double* ovals = vals0;
  int lev = 0;
  for (;;) {
    TW_G(ga)
    int parent, nout, nchild;
    if (!skip_first) {
      select_and_emit(sm, act, w, slot, oids, ocnt, ovals, nsl == 1 ? ro : TslwRoot{}, p0);
      TW_G(gb)
      if (nsl == 1 || lev == stop_lev) {  // the root, or a rank's top level (row-sharded path)
        TW_LV(lev, ga, gb, gb, gb)
        break;
      }
      // climb: the last child of the parent runs it
      if (cids) arrive += nsl;  // counters of this level's parents follow the previous level's
      parent = slot / arity, nout = (nsl + arity - 1) / arity;
      nchild = min(arity, nsl - parent * arity);
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atom_add_acq_rel_gpu(&arrive[parent], 1);  // releases this slot, acquires the others
      old = __shfl_sync(0xffffffffu, old, 0);
      TW_G(gc)
      if (old != nchild - 1) {
        TW_LV(lev + 100, ga, gb, gc, gc)
        break;
      }
      if (lane == 0) arrive[parent] = 0;  // every child has arrived: ready for the next panel
    } else {
      skip_first = false;
      parent = slot / arity, nout = (nsl + arity - 1) / arity;
      nchild = min(arity, nsl - parent * arity);
    }
    const bool first = cids == nullptr;
    cids = oids;
    cvals = ovals;
    oids = first ? idsN : oids + nsl * WW;
    ocnt = first ? cntN : ocnt + nsl;
    ovals = first ? valsN : ovals + (size_t)nsl * WW * WW;
    // children [parent*arity, +nchild): entry e of child ci -> tile row ci*16 + e, its ids and
    // (original) panel rows loaded in one pass (L2: written by other SMs in this launch)
    {
      const int ch = lane & 7;
#pragma unroll 8
      for (int i = 0; i < WR / 4; i++) {
        const int q = 4 * i + (lane >> 3), ci = q / WW, e = q % WW;
        const bool ok = ci < nchild;
        cp_async16_cg(sm.tile + q * TS + 2 * ch,
                      ok ? cvals + ((size_t)(parent * arity + ci) * WW + e) * WW + 2 * ch : cvals, ok ? 16 : 0);
      }
      cp_async_commit();
    }
    // rank = position in increasing-id order: the children cover increasing global row
    // ranges, so rank = ci*16 + (rank of the id within its child)
#pragma unroll
    for (int s = 0; s < RS; s++) {
      const int c = s * 32 + lane, ci = c / WW, e = c % WW, child = parent * arity + ci;
      const int v = ci < nchild ? __ldcg(cids + child * WW + e) : -1;  // -1: no entry
      const int id = v >= 0 ? v : INT_MAX;
      int rank = 0;
#pragma unroll
      for (int q = 0; q < WW; q++) {
        const int o = __shfl_sync(0xffffffffu, id, (lane & ~(WW - 1)) | q);
        rank += (o < id) || (o == id && q < e);
      }
      sm.sid[c] = id;
      sm.rank[c] = ci * WW + rank;
    }
    act = 0;
#pragma unroll
    for (int s = 0; s < RS; s++) act |= (sm.sid[s * 32 + lane] != INT_MAX ? 1u : 0u) << s;
    cp_async_wait_all();
    __syncwarp();
    TW_G(gd)
    TW_LV(lev, ga, ga, ga, gd)
    lev++;
    slot = parent;
    nsl = nout;
  }
}

// The tournament of one panel, all levels in one launch.  Warp = leaf (rows
// [leaf*128, leaf*128 + 128) of the local rows, their S_j rows from L's panel columns);
// the LAST child to finish a node runs the node (arrival counters, reset by the node's
// runner for the next panel), up to the root, which emits piv, U's diagonal block and
// 1/diag(U).  No launch per level, and the select code stays hot in the instruction cache.
// Slots: level 0 in ids0/cnt0, levels >= 1 packed in idsN/cntN (arrival counters alike).
__global__ void __launch_bounds__(32 * WPB)
tslw_tree_kernel(const double* __restrict__ Lb, int64_t ldl, int64_t rows, int64_t row0, int p0, int w,
                 const uint8_t* __restrict__ chosen, int* __restrict__ ids0, int* __restrict__ cnt0,
                 int* __restrict__ idsN, int* __restrict__ cntN, double* __restrict__ vals0,
                 double* __restrict__ valsN, int* __restrict__ arrive, int arity, int stop_lev, TslwRoot ro,
                 int start1) {
  extern __shared__ __align__(16) unsigned char raw[];
  WSel& sm = reinterpret_cast<WSel*>(raw)[warp_id()];
  pdl_trigger();
  pdl_wait();
  TW_T(t0)
  const int lane = lane_id();
  const int nleaves = (int)ceil_div<int64_t>(rows, WR);
  if (start1) {
    // the leaves were selected by the Schur kernel (tslw_schur_tma_kernel, slots ids0 / cnt0 /
    // vals0): warp = node of level 1, run as its last-arriving child would
    const int node = blockIdx.x * WPB + warp_id();
    if (node >= ceil_div(nleaves, arity)) return;
    tree_climb(sm, nleaves, node * arity, 0, nullptr, nullptr, ids0, cnt0, vals0, idsN, cntN, valsN, arrive, arity,
               stop_lev, ro, p0, w, true);
    return;
  }
  const int leaf = blockIdx.x * WPB + warp_id();
  if (leaf >= nleaves) return;
  const bool v16 = (ldl & 1) == 0 && (reinterpret_cast<uintptr_t>(Lb) & 15) == 0;
  const int64_t rb = (int64_t)leaf * WR;
  unsigned act = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int64_t r = rb + s * 32 + lane;
    sm.sid[s * 32 + lane] = r < rows ? (int)(row0 + r) : INT_MAX;
    sm.rank[s * 32 + lane] = s * 32 + lane;  // the leaf's rows are in increasing-id order
  }
  __syncwarp();
  stage_rows(sm, w, Lb, ldl, row0, p0, v16, false);  // in flight while the flags load
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int64_t r = rb + s * 32 + lane;
    act |= ((r < rows && !(chosen && chosen[r])) ? 1u : 0u) << s;
  }
  if (v16) {
    cp_async_wait_all();
    __syncwarp();
  }
  TW_T(t1)
  tree_climb(sm, nleaves, leaf, act, nullptr, nullptr, ids0, cnt0, vals0, idsN, cntN, valsN, arrive, arity, stop_lev,
             ro, p0, w, false);
  TW_T(t2)
  TW_T(t3)
  TW_REC(0, t0, t1, t2, t3)
}

// U rows [p0, p0+w) right of the panel: U[p0+t, c] = X[p_t, c] - sum_{k<p0} L[p_t, k] U[k, c]
// - sum_{t'<t} l_{t,t'} U[p0+t', c] (the oracle's elimination chain of the pivot row), with
// the in-panel multipliers l_{t,t'} recomputed from the winners' S_j rows by the same
// forward substitution (same chain as the select).  CTA: WW x 32 threads (row t, column).
constexpr int UR_C = 32, UR_K = 32;
__global__ void __launch_bounds__(WW * UR_C)
tslw_urows_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ Lb, int64_t ldl,
                  int64_t row0, int p0, int w, int n, const int64_t* __restrict__ piv, double* __restrict__ U,
                  const double* __restrict__ rd) {
  __shared__ double Lw[WW][UR_K + 1];
  __shared__ double Ut[UR_K][UR_C];
  __shared__ double P[WW][UR_C];
  __shared__ double lw[WW][WW + 1];
  __shared__ double Sb[WW][WW + 1];
  __shared__ double Ub[WW][WW + 1];
  __shared__ double rdb[WW];
  __shared__ int64_t prow[WW];
  pdl_trigger();
  pdl_wait();
  const int tx = threadIdx.x % UR_C, t = threadIdx.x / UR_C;
  const int c = p0 + w + blockIdx.x * UR_C + tx;
  if (threadIdx.x < WW) {
    prow[threadIdx.x] = threadIdx.x < w ? piv[p0 + threadIdx.x] - row0 : 0;
    rdb[threadIdx.x] = threadIdx.x < w ? rd[p0 + threadIdx.x] : 0.0;
  }
  {
    const int q = threadIdx.x % WW, k = threadIdx.x / WW;  // 512 threads cover 16 x 32
    if (k < WW) Ub[k][q] = (k < w && q < w) ? U[(int64_t)(p0 + k) * n + p0 + q] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < WW * WW) {
    const int tt = threadIdx.x / WW, q = threadIdx.x % WW;
    Sb[tt][q] = (tt < w && q < w) ? Lb[prow[tt] * ldl + p0 + q] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < w) {  // multipliers of winner t: S_j row -> substitution with U's block
    const int tt = threadIdx.x;
    double l[WW];
#pragma unroll
    for (int q = 0; q < WW; q++) l[q] = Sb[tt][q];
    subst_row_rl(l, tt, [&](int k, int q) { return Ub[k][q]; }, [&](int k) { return rdb[k]; });
#pragma unroll
    for (int q = 0; q < WW; q++) lw[tt][q] = l[q];
  }
  double acc = (t < w && c < n) ? X[prow[t] * ldx + c] : 0.0;
  for (int k0 = 0; k0 < p0; k0 += UR_K) {
    for (int e = threadIdx.x; e < WW * UR_K; e += blockDim.x) {
      const int tt = e / UR_K, kk = e - tt * UR_K;
      Lw[tt][kk] = (tt < w && k0 + kk < p0) ? Lb[prow[tt] * ldl + k0 + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < UR_K * UR_C; e += blockDim.x) {
      const int kk = e / UR_C, x = e - kk * UR_C, cc = p0 + w + blockIdx.x * UR_C + x;
      Ut[kk][x] = (k0 + kk < p0 && cc < n) ? U[(int64_t)(k0 + kk) * n + cc] : 0.0;
    }
    __syncthreads();
    const int kn = min(UR_K, p0 - k0);
    for (int kk = 0; kk < kn; kk++) acc = __fma_rn(-Lw[t][kk], Ut[kk][tx], acc);
    __syncthreads();
  }
  P[t][tx] = acc;
  __syncthreads();
  if (t == 0 && c < n) {
    double u[WW];
#pragma unroll
    for (int tt = 0; tt < WW; tt++) {
      if (tt < w) {
        double v = P[tt][tx];
#pragma unroll
        for (int q = 0; q < tt; q++) v = __fma_rn(-lw[tt][q], u[q], v);
        u[tt] = v;
        U[(int64_t)(p0 + tt) * n + c] = v;
      }
    }
  }
}

// Last panel: S -> L in place (forward substitution with U's diagonal block).
__global__ void __launch_bounds__(256)
tslw_lfinal_kernel(double* __restrict__ Lb, int64_t ldl, int64_t rows, int pl, int wl, int n,
                   const double* __restrict__ U, const double* __restrict__ rd) {
  __shared__ double Ub[WW][WW];
  __shared__ double rdp[WW];
  __shared__ double tile[256 * ST];
  pdl_trigger();
  pdl_wait();
  const int64_t rb = (int64_t)blockIdx.x * 256;
  // the CTA's 256 rows x wl columns, coalesced (16 threads per row)
  {
    const int c = threadIdx.x & 15;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const int q = (threadIdx.x >> 4) + 16 * j;
      const bool in = rb + q < rows && c < wl;
      cp_async8(tile + q * ST + c, in ? Lb + (rb + q) * ldl + pl + c : Lb, in ? 8 : 0);
    }
    cp_async_commit();
  }
  for (int e = threadIdx.x; e < WW * WW; e += blockDim.x) {
    const int k = e / WW, c = e - k * WW;
    Ub[k][c] = (k < wl && c < wl) ? U[(int64_t)(pl + k) * n + pl + c] : 0.0;
  }
  if (threadIdx.x < WW)
    rdp[threadIdx.x] = threadIdx.x >= wl ? 0.0
                       : rd ? rd[pl + threadIdx.x] : __ddiv_rn(1.0, U[(int64_t)(pl + threadIdx.x) * (n + 1)]);
  cp_async_wait_all();
  __syncthreads();
  double l[WW];
  double* row = tile + threadIdx.x * ST;
#pragma unroll
  for (int c = 0; c < WW; c++) l[c] = row[c];
  subst_row_rl(l, wl, [&](int k, int c) { return Ub[k][c]; }, [&](int k) { return rdp[k]; });
#pragma unroll
  for (int c = 0; c < WW; c++) row[c] = l[c];
  __syncthreads();
  {
    const int c = threadIdx.x & 15;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const int q = (threadIdx.x >> 4) + 16 * j;
      if (rb + q < rows && c < wl) Lb[(rb + q) * ldl + pl + c] = tile[q * ST + c];
    }
  }
}

// Pivot row t: L11 row t = its L row in columns < t, 1 on the diagonal, 0 right of it; the
// same values overwrite its L row (pivot rows take their L11 rows, oracle l_row).
// (Row-sharded: rows = this rank's row count; other ranks' pivot rows are skipped; L11 may be null.)
__global__ void tslw_fixup_kernel(double* __restrict__ Lb, int64_t ldl, int64_t row0, const int64_t* __restrict__ piv,
                                  int n, double* __restrict__ L11, int64_t rows) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int64_t r = piv[t] - row0;
  if (r < 0 || r >= rows) return;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double v = c < t ? Lb[r * ldl + c] : (c == t ? 1.0 : 0.0);
    if (L11) L11[(int64_t)t * n + c] = v;
    if (c >= t) Lb[r * ldl + c] = v;
  }
}

// Row-sharded TSLU (the warp contract): the current rows of the panel's winners that this
// rank owns, T[e][c - p0] = X[id_e, c] - sum_{k<p0} L[id_e, k] U[k, c] for c in [p0, n) (the
// fma chain of tslw_urows_kernel's first phase); 0 for winners owned by other ranks, so the
// all-reduced sum is every winner's row exactly.  CTA: 16 winners x 32 columns.
__global__ void __launch_bounds__(WW * 32)
tslw_owned_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ Lb, int64_t ldl,
                  int64_t rows, int64_t row0, const int* __restrict__ ids, int cnt, int p0, int n,
                  const double* __restrict__ U, double* __restrict__ T) {
  __shared__ double Lw[WW][33];
  __shared__ double Ut[32][32];
  __shared__ int64_t lr[WW];
  const int tx = threadIdx.x % 32, t = threadIdx.x / 32;
  const int c = p0 + blockIdx.x * 32 + tx;
  if (threadIdx.x < WW) {
    const int64_t r = threadIdx.x < cnt ? (int64_t)ids[threadIdx.x] - row0 : -1;
    lr[threadIdx.x] = (r >= 0 && r < rows) ? r : -1;
  }
  __syncthreads();
  const bool mine = t < cnt && lr[t] >= 0;
  double acc = (mine && c < n) ? X[lr[t] * ldx + c] : 0.0;
  for (int k0 = 0; k0 < p0; k0 += 32) {
    for (int e = threadIdx.x; e < WW * 32; e += blockDim.x) {
      const int tt = e / 32, kk = e % 32;
      Lw[tt][kk] = (lr[tt] >= 0 && tt < cnt && k0 + kk < p0) ? Lb[lr[tt] * ldl + k0 + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
      const int kk = e / 32, x = e % 32, cc = p0 + blockIdx.x * 32 + x;
      Ut[kk][x] = (k0 + kk < p0 && cc < n) ? U[(int64_t)(k0 + kk) * n + cc] : 0.0;
    }
    __syncthreads();
    const int kn = min(32, p0 - k0);
    for (int kk = 0; kk < kn; kk++) acc = __fma_rn(-Lw[t][kk], Ut[kk][tx], acc);
    __syncthreads();
  }
  if (t < cnt && c < n) T[(int64_t)t * (n - p0) + (c - p0)] = mine ? acc : 0.0;
}


// ------------------------------------------------------------------ exact GEPP mode
// One leaf holding every row (leaf_rows >= rows): the tournament of a
// panel is plain GEPP on all remaining rows (oracle gepp_select with one candidate set),
// i.e. exact partial pivoting with ties to the smallest row id.  One cooperative launch per
// panel, thread per row (grid-strided): each step t updates the working copy Sw of the
// panel's Schur values with step t-1 (the select's own ops: l = a * (1/pivot), a[c] =
// fma(-l, u[c], a[c])), then the grid finds the pivot in two atomic rounds -- the largest
// |a| bit pattern, then the smallest row among the rows attaining it -- and the owner
// publishes the pivot row.  Three grid barriers per step.
struct TslgScratch {
  unsigned long long gmax[WW];
  unsigned int gidx[WW];
  double prow[WW][WW];
  double r[WW];
};
__global__ void __launch_bounds__(256)
tslg_kernel(const double* __restrict__ Lb, int64_t ldl, double* __restrict__ Sw, int64_t rows, int64_t row0, int p0,
            int w, uint8_t* __restrict__ chosen, TslgScratch* sc, TslwRoot ro) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long bkey[8];
  __shared__ unsigned int bidx[8];
  __shared__ double up[WW];
  __shared__ double rprev;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = lane_id(), wq = warp_id();
  if (tid0 == 0) {
    for (int t = 0; t < WW; t++) {
      sc->gmax[t] = 0ull;
      sc->gidx[t] = 0xffffffffu;
    }
  }
  grid.sync();
  for (int t = 0; t < w; t++) {
    if (threadIdx.x < WW) up[threadIdx.x] = t > 0 ? sc->prow[t - 1][threadIdx.x] : 0.0;
    if (threadIdx.x == 0) rprev = t > 0 ? sc->r[t - 1] : 0.0;
    __syncthreads();
    unsigned long long best = 0;
    unsigned int bi = 0xffffffffu;
    for (int64_t r = tid0; r < rows; r += nthr) {
      if (__ldcg(chosen + r)) continue;  // set by another SM during this launch
      double v[WW];
      if (t == 0) {
#pragma unroll
        for (int c = 0; c < WW; c++) v[c] = c < w ? Lb[r * ldl + p0 + c] : 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < WW; c++) v[c] = Sw[r * WW + c];
        if (rprev != 0.0) {  // step t-1 was not a zero column (R#5 has no update)
          double l = 0.0;
#pragma unroll
          for (int c = 0; c < WW; c++)
            if (c == t - 1) l = __dmul_rn(v[c], rprev);
#pragma unroll
          for (int c = 0; c < WW; c++) {
            if (c == t - 1) v[c] = l;
            else if (c >= t) v[c] = __fma_rn(-l, up[c], v[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < WW; c++) Sw[r * WW + c] = v[c];
      double vt = 0.0;
#pragma unroll
      for (int c = 0; c < WW; c++)
        if (c == t) vt = v[c];
      const unsigned long long key = (unsigned long long)__double_as_longlong(vt) & 0x7fffffffffffffffull;
      if (key > best || bi == 0xffffffffu) {  // rows ascend: the first of equal keys is kept
        best = key;
        bi = (unsigned int)r;
      }
    }
    // block maximum of the key, then the grid's
    unsigned long long k = best;
    for (int o = 16; o; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, k, o);
      k = x > k ? x : k;
    }
    if (lane == 0) bkey[wq] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); q++) m = bkey[q] > m ? bkey[q] : m;
      atomicMax(&sc->gmax[t], m);
    }
    grid.sync();
    // the smallest row attaining the maximum (ties -> smallest id, R#4)
    const unsigned long long gm = sc->gmax[t];
    unsigned int cand = (bi != 0xffffffffu && best == gm) ? bi : 0xffffffffu;
    for (int o = 16; o; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
    if (lane == 0) bidx[wq] = cand;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int m = 0xffffffffu;
      for (int q = 0; q < (int)(blockDim.x >> 5); q++) m = min(m, bidx[q]);
      if (m != 0xffffffffu) atomicMin(&sc->gidx[t], m);
    }
    grid.sync();
    const unsigned int p = sc->gidx[t];
    if (tid0 == 0) {  // publish the pivot row (after t updates), 1/pivot; root outputs
      const bool zero = gm == 0 || p == 0xffffffffu;
      const unsigned int pp = p == 0xffffffffu ? 0u : p;
      double pv = 0.0;
      for (int c = 0; c < WW; c++) {
        const double x = __ldcg(Sw + (int64_t)pp * WW + c);
        sc->prow[t][c] = x;
        if (c == t) pv = x;
      }
      const double rr = zero ? 0.0 : __drcp_rn(pv);
      sc->r[t] = rr;
      chosen[pp] = 1;
      ro.piv[p0 + t] = row0 + pp;
      ro.rd[p0 + t] = rr;
      if (zero) report(ro.status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + t);
      for (int c = t; c < w; c++) ro.U[(int64_t)(p0 + t) * ro.n + p0 + c] = __ldcg(Sw + (int64_t)pp * WW + c);
    }
    grid.sync();
  }
}

// The warp kernels use 16-column panels: the contract's panel must be 16, or n when n < 16.
bool tslw_cfg(const rlhc_tslu_cfg& c, int64_t m, int64_t n) {
  if (!(c.panel == WW || (c.panel == n && n < WW))) return false;
  if (c.leaf_rows >= m && c.arity >= 2) return true;  // exact GEPP mode (one leaf)
  return c.leaf_rows == WR && c.arity >= 2 && c.arity * WW <= WR;
}
bool tslg_cfg(const rlhc_tslu_cfg& c, int64_t m, int64_t n) { return tslw_cfg(c, m, n) && c.leaf_rows >= m; }

size_t tslw_slots(int64_t rows) { return (size_t)ceil_div<int64_t>(rows, WR); }

// PX = LU on rows x n (global ids row0 + local row).  Lb (rows x n, ldl) receives L in
// original row order (pivot rows: their L11 rows); ids/cnt: two slot buffers of
// tslw_slots(rows) * 16 ids and counts; chosen: rows bytes; rd: 1/diag(U).
size_t tslg_ws_bytes(int64_t rows) { return (size_t)rows * WW * sizeof(double) + sizeof(TslgScratch) + 256; }

// The row-sharded path's local tournament (rlhc_tslu_reduce under the warp contract): the
// tree kernel on this rank's rows of the panel source `src` (current panel values, columns
// [p0, p0+w)), every local level down to ONE slot, no root outputs; the top slot (ids,
// count, the winners' panel rows) is copied to out_*.  cnt[1] holds the packed counts of the
// levels >= 1 followed by their arrival counters.
cudaError_t run_tslw_local_tree(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                                const uint8_t* chosen, int arity, int stop_lev, int* ids[2], int* cnt[2],
                                double* vals[2], int* out_ids, int* out_cnt, double* out_vals, cudaStream_t st) {
  cudaError_t e;
  const int nleaves = (int)tslw_slots(rows);
  // packed slots of the levels >= 1; offset and size of the output level (the root, or
  // level stop_lev when this rank's rows hold several complete subtrees)
  size_t above = 0, top = 0;
  int lev = 0, nout = nleaves;
  for (int ns = nleaves; ns > 1 && lev != stop_lev; ns = ceil_div(ns, arity)) {
    top = above;
    above += ceil_div(ns, arity);
    lev++;
    nout = ceil_div(ns, arity);
  }
  int* arrive = cnt[1] + above;
  if (above && (e = cudaMemsetAsync(arrive, 0, above * sizeof(int), st))) return e;
  static DevFlags attr;
  if ((e = smem_attr(attr, tslw_tree_kernel, 227 * 1024))) return e;
  note_launch();
  e = launch_pdl(tslw_tree_kernel, dim3(ceil_div(nleaves, WPB)), dim3(32 * WPB), WPB * sizeof(WSel), st, src, lds,
                 rows, row0, p0, w, chosen, ids[0], cnt[0], ids[1], cnt[1], vals[0], vals[1], arrive, arity,
                 stop_lev, TslwRoot{}, 0);
  if (e) return e;
  const int* tid = lev == 0 ? ids[0] : ids[1] + top * WW;
  const int* tcnt = lev == 0 ? cnt[0] : cnt[1] + top;
  const double* tval = lev == 0 ? vals[0] : vals[1] + top * WW * WW;
  if ((e = cudaMemcpyAsync(out_ids, tid, (size_t)nout * WW * sizeof(int), cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(out_cnt, tcnt, (size_t)nout * sizeof(int), cudaMemcpyDeviceToDevice, st))) return e;
  return cudaMemcpyAsync(out_vals, tval, (size_t)nout * WW * WW * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

// The row-sharded path's fused panel: this rank's Schur complement of panel p0 with its leaves
// selected inside the TMA Schur kernel (as run_tslw does), then the rank's tournament levels
// >= 1 up to stop_lev (-1: its root) in one launch, the top level's slots copied to out_*.
// *fused = false: the TMA kernel is not available for these buffers and nothing was launched.
// status (nullable): non-finite elements of X's panel columns reported as ENONFINITE(INPUT,
// row * n + column), as the single-process pipeline's folded input check.
cudaError_t run_tslw_schur_local_tree(const double* X, int64_t ldx, double* Lb, int64_t ldl, int64_t rows,
                                      int64_t row0, int p0, int w, int n, const double* U, const uint8_t* chosen,
                                      int arity, int stop_lev, int* ids[2], int* cnt[2], double* vals[2],
                                      int* out_ids, int* out_cnt, double* out_vals, unsigned long long* status,
                                      cudaStream_t st, bool* fused) {
  *fused = false;
  bool done = false, leaves_done = false;
  cudaError_t e = launch_schur_tma(X, ldx, Lb, ldl, rows, p0, w, n, U, nullptr, status, chosen, ids[0], cnt[0],
                                   vals[0], row0, st, &done, &leaves_done);
  if (e || !done) return e;
  *fused = true;
  if (!leaves_done)  // (one leaf, or no room for the select warps' buffers): the plain local tree
    return run_tslw_local_tree(Lb, ldl, rows, row0, p0, w, chosen, arity, stop_lev, ids, cnt, vals, out_ids,
                               out_cnt, out_vals, st);
  const int nleaves = (int)tslw_slots(rows);
  size_t above = 0, top = 0;
  int lev = 0, nout = nleaves;
  for (int ns = nleaves; ns > 1 && lev != stop_lev; ns = ceil_div(ns, arity)) {
    top = above;
    above += ceil_div(ns, arity);
    lev++;
    nout = ceil_div(ns, arity);
  }
  if (lev > 0) {
    int* arrive = cnt[1] + above;
    if ((e = cudaMemsetAsync(arrive, 0, above * sizeof(int), st))) return e;
    static DevFlags attr;
    if ((e = smem_attr(attr, tslw_tree_kernel, 227 * 1024))) return e;
    note_launch();
    e = launch_pdl(tslw_tree_kernel, dim3(ceil_div(ceil_div(nleaves, arity), WPB)), dim3(32 * WPB),
                   WPB * sizeof(WSel), st, (const double*)Lb, ldl, rows, row0, p0, w, chosen, ids[0], cnt[0], ids[1],
                   cnt[1], vals[0], vals[1], arrive, arity, stop_lev, TslwRoot{}, 1);
    if (e) return e;
  }
  const int* tid = lev == 0 ? ids[0] : ids[1] + top * WW;
  const int* tcnt = lev == 0 ? cnt[0] : cnt[1] + top;
  const double* tval = lev == 0 ? vals[0] : vals[1] + top * WW * WW;
  if ((e = cudaMemcpyAsync(out_ids, tid, (size_t)nout * WW * sizeof(int), cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(out_cnt, tcnt, (size_t)nout * sizeof(int), cudaMemcpyDeviceToDevice, st))) return e;
  return cudaMemcpyAsync(out_vals, tval, (size_t)nout * WW * WW * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

// per host thread and device: the look-ahead's side stream and its fork / join events
struct LookAhead {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static cudaError_t look_ahead_streams(LookAhead** out) {
  static thread_local LookAhead per_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  LookAhead& la = per_dev[dev];
  if (!la.side) {
    if ((e = cudaStreamCreateWithFlags(&la.side, cudaStreamNonBlocking))) return e;
    if ((e = cudaEventCreateWithFlags(&la.fork, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&la.join, cudaEventDisableTiming))) return e;
  }
  *out = &la;
  return cudaSuccess;
}

// Panels are grouped by kTslwGroup (64 columns): at the start of group g >= 1 the last panel's
// Schur values become L (tslw_lfinal_kernel) and ONE product B = X[:, group] - L[:, :P0]
// U[:P0, group] (tsgemm.cu, TMA-fed DMMA, the fma chain in increasing k) goes into Lb's group
// columns; the group's first panel is then B's first 16 columns (no Schur kernel), the others
// continue the chain over the group's earlier columns only.  Every L column is read from HBM
// once per group instead of once per panel (cfg5: 395 -> ~300 GB), and the bulk runs on the
// tensor pipe at 16 flops per byte.  Measured at cfg5 (profiles/r02_launches_cfg5_*.txt): the
// bulk ran at 48 % of the DMMA peak (short K for the first groups, each tile's X loads
// exposed) and the in-group Schur kernels kept 3.3 ms each, so the LU went 104 -> 116 ms:
// OFF by default; RLHC_LU_GROUP=1 (measurement knob) enables it.
cudaError_t run_tslw(const double* X, int64_t ldx, int64_t rows, int64_t row0, int n, int arity, double* Lb,
                     int64_t ldl, int64_t* piv, double* U, double* L11, double* rd, double* lw, uint8_t* chosen,
                     int* ids[2], int* cnt[2], double* vals[2], unsigned long long* status, bool check_input,
                     cudaStream_t st, void* gepp_ws, double* bpack, const TslwPanelHook* hook) {
  (void)lw;
  static const bool group_on = [] { const char* e = getenv("RLHC_LU_GROUP"); return e && atoi(e) != 0; }();
  const bool grouped = group_on && bpack && !gepp_ws;
  // look-ahead (RLHC_LU_LOOKAHEAD=1, measurement knob): panel p+1's Schur complement minus its
  // last 16 terms runs on a side stream while panel p's tournament -- a latency chain that
  // leaves HBM idle -- climbs its tree.  Measured slower (cfg5 TSLU 106 -> 128 ms, cfg3 3.2 ->
  // 3.5 ms): the tree's leaf wave fills every SM, so the two kernels only slow each other,
  // and the split adds a write and a read of the partial panel.  Off by default.
  static const bool look_on = [] { const char* e = getenv("RLHC_LU_LOOKAHEAD"); return e && atoi(e) != 0; }();
  LookAhead* la = nullptr;
  if (look_on && !grouped && !gepp_ws) {
    if (cudaError_t e0 = look_ahead_streams(&la)) return e0;
  }
  const bool look = la != nullptr;
  double* Sw = gepp_ws ? reinterpret_cast<double*>(gepp_ws) : nullptr;  // exact GEPP mode (one leaf)
  TslgScratch* gsc = gepp_ws ? reinterpret_cast<TslgScratch*>(reinterpret_cast<char*>(gepp_ws) +
                                                               (((size_t)rows * WW * sizeof(double) + 255) & ~(size_t)255))
                             : nullptr;
  cudaError_t e;
  const int nleaves = (int)tslw_slots(rows);
  // slots: level 0 in ids[0]/cnt[0]; levels >= 1 packed in ids[1]/cnt[1]; the arrival
  // counters of levels >= 1 follow the packed counts in cnt[1]
  size_t above = 0;
  for (int ns = nleaves; ns > 1; ns = ceil_div(ns, arity)) above += ceil_div(ns, arity);
  int* arrive = cnt[1] + above;
  if ((e = cudaMemsetAsync(chosen, 0, (size_t)rows, st))) return e;
  if ((e = cudaMemsetAsync(U, 0, (size_t)n * n * sizeof(double), st))) return e;
  if ((e = cudaMemsetAsync(arrive, 0, above * sizeof(int), st))) return e;
  static DevFlags attr_t, attr_s;
  if ((e = smem_attr(attr_t, tslw_tree_kernel, 227 * 1024))) return e;
  if ((e = smem_attr(attr_s, tslw_schur_dmma_kernel, (int)sizeof(SchurDSmem)))) return e;
  const TslwRoot root{U, piv, rd, nullptr, chosen, status, row0, n};
  static const bool pair_on = [] { const char* e = getenv("RLHC_LU_PAIR"); return !e || atoi(e) != 0; }();
  static const int pair_min = [] { const char* e = getenv("RLHC_LU_PAIR_MIN"); return e ? std::max(2, atoi(e)) : 6; }();
  // RLHC_LU_PAIR_SPLIT=f (percent, measurement knob): the even panel j's partial for panel j+1
  // covers only L chunks [0, round(f j / 100)); the odd panel streams the rest (same chain order)
  static const int pair_split = [] { const char* e = getenv("RLHC_LU_PAIR_SPLIT"); return e ? atoi(e) : 100; }();
  bool prev_pair = false;  // the previous panel's kernel left this panel's partial in Lb
  int split = -1;          // chunks the partial covers (-1: all)
  int pl = 0, wl = 0;
  for (int p0 = 0; p0 < n; p0 += WW) {
    const int w = std::min(WW, n - p0);
    bool leaves_done = false;  // the Schur kernel selected this panel's leaves
    const int P0 = grouped ? p0 - p0 % kTslwGroup : 0;  // start of this panel's group
    if (grouped && p0 >= kTslwGroup && p0 == P0) {
      // new group: S of the last panel -> L, then B = X[:, group] - L[:, :P0] U[:P0, group]
      note_launch();
      e = launch_pdl(tslw_lfinal_kernel, dim3((unsigned)ceil_div<int64_t>(rows, 256)), dim3(256), 0, st, Lb, ldl,
                     rows, p0 - WW, WW, n, (const double*)U, (const double*)rd);
      if (e) return e;
      e = launch_ts_gemm_checked(X + P0, ldx, Lb + P0, ldl, Lb, ldl, U + P0, n, rows, P0, std::min(kTslwGroup, n - P0),
                                 bpack, check_input ? status : nullptr, n, P0, st);
      if (e) return e;
    } else if (look && p0 >= 2 * WW) {
      // the look-ahead's second half: wait for this panel's bulk (pre-only, side stream), then
      // S_{p-1} -> L_{p-1} and the last 16 terms (k = p0-16 .. p0-1), from the partial in Lb
      if ((e = cudaStreamWaitEvent(st, la->join, 0))) return e;
      note_launch();
      e = launch_pdl(tslw_schur_dmma_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SD_M)), dim3(256),
                     sizeof(SchurDSmem), st, X, ldx, Lb, ldl, rows, p0, w, n, (const double*)U, (const double*)rd,
                     (unsigned long long*)nullptr, (const double*)Lb, ldl, p0 - WW, 0);
      if (e) return e;
    } else {
      bool done = false;
      if (!grouped && !look) {
        // panel pairs (RLHC_LU_PAIR, default on): an even panel p >= 2 also forms the next
        // panel's partial Schur complement from the same L chunks; the odd panel after it
        // starts from that partial (mode 2) and re-reads no L chunk
        const int pidx = p0 / WW, np = ceil_div(n, WW);
        int mode = 0, w2 = 0;
        if (pair_on && pidx >= pair_min && pidx % 2 == 0 && pidx + 1 < np) {
          mode = 1;
          w2 = std::min(WW, n - p0 - WW);
          split = pair_split >= 100 ? -1 : std::max(0, std::min(pidx, (pair_split * pidx + 50) / 100));
        } else if (prev_pair) {
          mode = 2;
        }
        e = launch_schur_tma(X, ldx, Lb, ldl, rows, p0, w, n, U, rd, check_input ? status : nullptr, chosen,
                             Sw ? nullptr : ids[0], cnt[0], vals[0], row0, st, &done, &leaves_done, mode, w2,
                             mode ? split : -1);
        if (e) return e;
        prev_pair = done && mode == 1;
      }
      if (!done) note_launch();
      e = done ? cudaSuccess
        : p0 ? launch_pdl(tslw_schur_dmma_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SD_M)), dim3(256),
                          sizeof(SchurDSmem), st, X, ldx, Lb, ldl, rows, p0, w, n, (const double*)U,
                          (const double*)rd, check_input ? status : nullptr, (const double*)(P0 ? Lb : X),
                          P0 ? ldl : ldx, P0, 0)
             : launch_pdl(tslw_schur0_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SR)), dim3(SR), 0, st, X, ldx,
                          Lb, ldl, rows, w, n, check_input ? status : nullptr);
      if (e) return e;
    }
    if (hook) {
      if ((e = hook->after_schur(hook->ctx, p0 / WW, ceil_div(n, WW), st))) return e;
    }
    if (look && p0 + WW < n && p0 + WW >= 2 * WW) {
      // look-ahead: the next panel's bulk X[:, q] - L[:, :p0] U[:p0, q] (every term but the
      // last 16; L[:, :p0] is final now) on the side stream, overlapping this panel's
      // tournament, into the next panel's columns of Lb
      const int q0 = p0 + WW, wq = std::min(WW, n - q0);
      if ((e = cudaEventRecord(la->fork, st))) return e;
      if ((e = cudaStreamWaitEvent(la->side, la->fork, 0))) return e;
      note_launch();
      e = launch_pdl(tslw_schur_dmma_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SD_M)), dim3(256),
                     sizeof(SchurDSmem), la->side, X, ldx, Lb, ldl, rows, q0, wq, n, (const double*)U,
                     (const double*)rd, check_input ? status : nullptr, X, ldx, 0, 1);
      if (e) return e;
      if ((e = cudaEventRecord(la->join, la->side))) return e;
    }
    if (Sw) {  // exact GEPP: one cooperative launch per panel
      // co-resident grid of the current device (SM count and occupancy queried per call: a
      // MIG slice or another device may have fewer SMs than a full B200)
      int dev = 0, sms = 0, per_sm = 0;
      if ((e = cudaGetDevice(&dev))) return e;
      if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tslg_kernel, 256, 0))) return e;
      const int gridg = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, 256),
                                                                    (int64_t)sms * std::max(per_sm, 1)));
      const double* Lbc = Lb;
      int p0v = p0, wv = w;
      int64_t rowsv = rows, row0v = row0, ldlv = ldl;
      TslwRoot rootv = root;
      void* args[] = {(void*)&Lbc, (void*)&ldlv, (void*)&Sw, (void*)&rowsv, (void*)&row0v, (void*)&p0v, (void*)&wv,
                      (void*)&chosen, (void*)&gsc, (void*)&rootv};
      note_launch();
      e = cudaLaunchCooperativeKernel((const void*)tslg_kernel, dim3(gridg), dim3(256), args, 0, st);
      if (e) return e;
    } else {
      note_launch();
      const int nwarps = leaves_done ? ceil_div(nleaves, arity) : nleaves;  // leaves_done: from level 1
      e = launch_pdl(tslw_tree_kernel, dim3(ceil_div(nwarps, WPB)), dim3(32 * WPB), WPB * sizeof(WSel), st,
                     (const double*)Lb, ldl, rows, row0, p0, w, (const uint8_t*)(p0 ? chosen : nullptr), ids[0],
                     cnt[0], ids[1], cnt[1], vals[0], vals[1], arrive, arity, -1, root, leaves_done ? 1 : 0);
      if (e) return e;
    }
    if (p0 + w < n) {
      note_launch();
      e = launch_pdl(tslw_urows_kernel, dim3(ceil_div(n - p0 - w, UR_C)), dim3(WW * UR_C), 0, st, X, ldx,
                     (const double*)Lb, ldl, row0, p0, w, n, (const int64_t*)piv, U, (const double*)rd);
      if (e) return e;
    }
    pl = p0;
    wl = w;
  }
  note_launch();
  e = launch_pdl(tslw_lfinal_kernel, dim3((unsigned)ceil_div<int64_t>(rows, 256)), dim3(256), 0, st, Lb, ldl, rows, pl,
                 wl, n, (const double*)U, (const double*)rd);
  if (e) return e;
  note_launch();
  return launch_pdl(tslw_fixup_kernel, dim3(n), dim3(128), 0, st, Lb, ldl, row0, (const int64_t*)piv, n, L11, rows);
}

// ------------------------------------------------------------------ row-sharded TSLU blocks
cudaError_t launch_tslw_schur(const double* X, int64_t ldx, double* Lb, int64_t ldl, int64_t rows, int p0, int w, int n,
                              const double* U, cudaStream_t st) {
  if (p0 > 0) {  // the TMA pipeline (same chain per element, so the same bits), leaves not fused
    bool done = false, leaves_done = false;
    cudaError_t e = launch_schur_tma(X, ldx, Lb, ldl, rows, p0, w, n, U, nullptr, nullptr, nullptr, nullptr, nullptr,
                                     nullptr, 0, st, &done, &leaves_done);
    if (e || done) return e;
  }
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, tslw_schur_dmma_kernel, (int)sizeof(SchurDSmem))) return e;
  note_launch();
  if (p0 == 0)
    return launch_pdl(tslw_schur0_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SR)), dim3(SR), 0, st, X, ldx, Lb,
                      ldl, rows, w, n, (unsigned long long*)nullptr);
  return launch_pdl(tslw_schur_dmma_kernel, dim3((unsigned)ceil_div<int64_t>(rows, SD_M)), dim3(256),
                    sizeof(SchurDSmem), st, X, ldx, Lb, ldl, rows, p0, w, n, U, (const double*)nullptr,
                    (unsigned long long*)nullptr, X, ldx, 0, 0);
}

cudaError_t launch_tslw_owned(const double* X, int64_t ldx, const double* Lb, int64_t ldl, int64_t rows, int64_t row0,
                              const int* ids, int cnt, int p0, int n, const double* U, double* T, cudaStream_t st) {
  note_launch();
  tslw_owned_kernel<<<ceil_div(n - p0, 32), WW * 32, 0, st>>>(X, ldx, Lb, ldl, rows, row0, ids, cnt, p0, n, U, T);
  return cudaGetLastError();
}

cudaError_t launch_tslw_finish(double* Lb, int64_t ldl, int64_t rows, int64_t row0, int n, const double* U,
                               const int64_t* piv, cudaStream_t st) {
  const int pl = ((n - 1) / WW) * WW, wl = n - pl;
  note_launch();
  cudaError_t e = launch_pdl(tslw_lfinal_kernel, dim3((unsigned)ceil_div<int64_t>(rows, 256)), dim3(256), 0, st, Lb,
                             ldl, rows, pl, wl, n, U, (const double*)nullptr);
  if (e) return e;
  note_launch();
  return launch_pdl(tslw_fixup_kernel, dim3(n), dim3(128), 0, st, Lb, ldl, row0, piv, n, (double*)nullptr, rows);
}

}  // namespace rlhc
