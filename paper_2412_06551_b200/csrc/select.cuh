// select.cuh -- the GEPP "select" of one tournament node (R#4-R#5), used by the
// leaf and node kernels of tslu.cu.
//
// Layout: CTA = NW warps, R = 32*RS candidate rows, panel width W, CW = W/NW columns per
// warp assigned ROUND-ROBIN: warp q owns panel columns {q + NW k : k < CW}; lane l holds
// rows {l + 32 s : s < RS}, so a[s][k] = row (l + 32 s), column q + NW k.
//
// Pipeline over per-step mbarriers (no CTA-wide barrier inside the elimination).  Step t
// pivots on column t, owned by warp t % NW at local column K = t / NW.  Every warp, for
// every step t:
//   * waits for step t-1's publication (mbarrier t-1), reads its multipliers and pivot row;
//   * if it owns step t: applies step t-1 to column K first, publishes the updated column,
//     finds the pivot (warp-local max |a[.][K]|, ties -> smallest global id), publishes
//     r = 1/pivot and arrives on mbarrier t, then applies step t-1 to its columns > K;
//   * otherwise applies step t-1 to its columns >= K.
// Consecutive steps have different owners, so the critical path per step is one column
// update + one argmax; the bulk update runs in the shadow of the next owner's pivot search.
// Every warp forms the multipliers l = col * r itself (the oracle's IEEE product).  Every
// step's column stays in shared memory (W x R doubles): no slot is reused, a producer never
// waits for a consumer.  The per-element fma chain (increasing step order) is the oracle's,
// so the pivots are bit-identical to gepp_select.
#pragma once
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

#ifdef RLHC_SEL_TRACE
// probe builds only (tools/probe/psel.cu): per-step timestamps in shared memory
#define SEL_TRACE(idx) \
  if (lane_id() == 0) sm.trace[(idx)] = clock64();
#else
#define SEL_TRACE(idx)
#endif

template <int W, int NW, int RS>
struct SelSmem {
  double col[W][32 * RS];      // pivot column of step t after its update (candidate s*32 + lane)
  double col_pad[32 * RS];     // with col: the candidate staging area R x (W + 1) before the select
  double r[W];                 // |1 / pivot| of step t
  unsigned long long bar[W];   // mbarrier of step t (32 arrivals: the owner warp)
  int prow[W];                 // candidate index of the pivot row of step t
  int zero[W];                 // 1: zero pivot column at step t (R#5: no update); -1: pivot < 0
  int out_src[W];              // candidate index of the winner of step t (filled after the loop)
  int out_id[W];               // its global id
  int cgid[32 * RS];           // global id of candidate s*32 + lane (node kernel: entry ids first)
  int perm[32 * RS];           // node kernel: candidate index -> loaded entry (-1: none)
  double* Uout;                // root emission (single panel): U rows, ld = ldu; else null
  int ldu;
#ifdef RLHC_SEL_TRACE
  long long trace[(W + 1) * 32];
#endif
};

// a[pslot][k] (k compile-time, pslot warp-uniform): log2(RS)-level mux, no branches
template <int RS, int CW>
RLHC_DEV double sel_mux(const double (&a)[RS][CW], int k, int pslot) {
  double m[RS];
#pragma unroll
  for (int s = 0; s < RS; s++) m[s] = a[s][k];
#pragma unroll
  for (int b = 1; b < RS; b <<= 1) {
    const bool p = (pslot & b) != 0;
#pragma unroll
    for (int s = 0; s + b < RS; s += 2 * b) m[s] = p ? m[s + b] : m[s];
  }
  return m[0];
}

// u[k] = a[pslot][k] in lane `plane` for k in [K0, CW) (not yet broadcast: sel_bcast).
// Only the pivot lane runs the switch: one branch instead of CW muxes.
#define RLHC_SEL_CASE(S)                                   \
  case S:                                                  \
    if constexpr (S < RS) {                                \
      _Pragma("unroll") for (int k = K0; k < CW; k++) u[k] = a[S][k]; \
    }                                                      \
    break;
template <int RS, int CW, int K0>
RLHC_DEV void sel_row(const double (&a)[RS][CW], int pslot, int plane, double (&u)[CW]) {
  static_assert(RS <= 16, "sel_row handles up to 16 slots");
  if (lane_id() == plane) {
    switch (pslot) {
      RLHC_SEL_CASE(0) RLHC_SEL_CASE(1) RLHC_SEL_CASE(2) RLHC_SEL_CASE(3)
      RLHC_SEL_CASE(4) RLHC_SEL_CASE(5) RLHC_SEL_CASE(6) RLHC_SEL_CASE(7)
      RLHC_SEL_CASE(8) RLHC_SEL_CASE(9) RLHC_SEL_CASE(10) RLHC_SEL_CASE(11)
      RLHC_SEL_CASE(12) RLHC_SEL_CASE(13) RLHC_SEL_CASE(14) RLHC_SEL_CASE(15)
      default: break;
    }
  }
}
#undef RLHC_SEL_CASE
template <int CW, int K_LO, int K_HI>
RLHC_DEV void sel_bcast(double (&u)[CW], int plane) {
#pragma unroll
  for (int k = K_LO; k < K_HI; k++) u[k] = __shfl_sync(0xffffffffu, u[k], plane);
}

// a[.][k] -= l * u[k] for k in [K_LO, K_HI)
template <int RS, int CW, int K_LO, int K_HI>
RLHC_DEV void sel_update(double (&a)[RS][CW], const double (&l)[RS], const double (&u)[CW]) {
#pragma unroll
  for (int s = 0; s < RS; s++) {
#pragma unroll
    for (int k = K_LO; k < K_HI; k++) a[s][k] = __fma_rn(-l[s], u[k], a[s][k]);
  }
}

// Pivot search on column K and publication of step t (owner warp only).  Publishes the
// updated column itself (before the search), |1/pivot| and the pivot's sign; every warp
// forms l = col * r, the same IEEE product as the oracle.
//
// Candidates are held in increasing global-id order (candidate index s*32 + lane: the leaf
// loads rows in order, the node kernel sorts its candidates), so "the smallest global id
// among the rows attaining the maximum" (R#4) is the first candidate index attaining it:
// one ballot per slot, no id reduction.  The maximum of the |a| bit patterns (sign bit
// cleared: a total order on non-negative doubles that also ranks NaN, which the trailing
// matrix can hold after a rank deficiency) is taken on the 32-bit halves: the high words,
// then the low words among the candidates that attain the high maximum.
template <int W, int NW, int RS, int K>
RLHC_DEV void sel_pivot(const double (&a)[RS][W / NW], unsigned act, int t, SelSmem<W, NW, RS>& sm) {
  const int lane = lane_id();
#pragma unroll
  for (int s = 0; s < RS; s++) sm.col[t][s * 32 + lane] = a[s][K];
  int hi[RS];
  unsigned lo[RS], negm = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const int h = __double2hiint(a[s][K]);
    hi[s] = ((act >> s) & 1u) ? (h & 0x7fffffff) : -1;
    lo[s] = (unsigned)__double2loint(a[s][K]);
    negm |= (a[s][K] < 0.0 ? 1u : 0u) << s;
  }
  int mh = hi[0];
#pragma unroll
  for (int s = 1; s < RS; s++) mh = max(mh, hi[s]);
  SEL_TRACE(t * 32 + 18)
  mh = __reduce_max_sync(0xffffffffu, mh);
  SEL_TRACE(t * 32 + 19)
  unsigned ml = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) ml = max(ml, hi[s] == mh ? lo[s] : 0u);
  ml = __reduce_max_sync(0xffffffffu, ml);
  SEL_TRACE(t * 32 + 20)
  const long long gb = (long long)(((unsigned long long)(unsigned)mh << 32) | ml);
  // |1/pivot| (independent of which row attains it), branch-free so that it overlaps the
  // ballots below; exponents outside its window take __drcp_rn after them
  const double pabs = __longlong_as_double(gb);
  double rabs = rcp_newton(pabs);
  // smallest candidate index s*32 + lane attaining the maximum (an active candidate always
  // does): this lane's first matching slot, then one warp minimum
  unsigned mm = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) mm |= (hi[s] == mh && lo[s] == ml ? 1u : 0u) << s;
  const int pidx = __reduce_min_sync(0xffffffffu, mm ? (__ffs(mm) - 1) * 32 + lane : INT_MAX);
  SEL_TRACE(t * 32 + 21)
  if (!rcp_newton_ok(mh)) rabs = rcp_slow(pabs);  // warp-uniform, rare
  const bool neg = (negm >> (pidx >> 5)) & 1u;    // meaningful in the pivot's lane
  if (lane == (pidx & 31)) {
    sm.prow[t] = pidx;
    sm.r[t] = rabs;
    sm.zero[t] = gb == 0 ? 1 : (neg ? -1 : 0);  // 1: zero column (R#5); -1: negative pivot
  }
  SEL_TRACE(t * 32 + 22)
  mbar_arrive(&sm.bar[t]);
  if (lane == (pidx & 31) && sm.Uout)  // root emission: U(t, t) = the pivot (|pivot| and sign)
    sm.Uout[(int64_t)t * sm.ldu + t] = neg ? -pabs : pabs;
}

// Step t (local pivot column K of warp t % NW): consume step t-1, own step t if mine.
template <int W, int NW, int RS, int K>
RLHC_DEV void sel_step(double (&a)[RS][W / NW], unsigned& act, int t, bool own,
                       SelSmem<W, NW, RS>& sm) {
  constexpr int CW = W / NW;
  const int lane = lane_id();
  bool upd = false;
  int pslot = 0, plane = 0;
  double l[RS], u[CW];
  if (t > 0) {
    mbar_wait(&sm.bar[t - 1], 0);
    SEL_TRACE(t * 32 + warp_id() * 2)
    const int prow = sm.prow[t - 1];
    pslot = prow >> 5;
    plane = prow & 31;
    const int zf = sm.zero[t - 1];
    upd = zf != 1;
    if (upd) {
      const double r = zf < 0 ? -sm.r[t - 1] : sm.r[t - 1];  // drcp(-x) == -drcp(x)
#pragma unroll
      for (int s = 0; s < RS; s++) l[s] = __dmul_rn(sm.col[t - 1][s * 32 + lane], r);
    }
    if (lane == plane) act &= ~(1u << pslot);
  }
  if (own) {
    if (upd) {
      const double uk = __shfl_sync(0xffffffffu, sel_mux<RS, CW>(a, K, pslot), plane);
      u[K] = uk;
#pragma unroll
      for (int s = 0; s < RS; s++) a[s][K] = __fma_rn(-l[s], uk, a[s][K]);
    }
    SEL_TRACE(t * 32 + 16)
    sel_pivot<W, NW, RS, K>(a, act, t, sm);
    SEL_TRACE(t * 32 + 17)
    if (upd) {
      sel_row<RS, CW, K + 1>(a, pslot, plane, u);
      sel_bcast<CW, K + 1, CW>(u, plane);
      sel_update<RS, CW, K + 1, CW>(a, l, u);
    }
  } else if (upd) {
#ifndef RLHC_SEL_NOCONS
    sel_row<RS, CW, K>(a, pslot, plane, u);
    sel_bcast<CW, K, CW>(u, plane);
    sel_update<RS, CW, K, CW>(a, l, u);
#endif
  }
  // root emission: U(t-1, c) for this warp's columns c > t-1 = the pivot row's values after
  // t-1 eliminations (the oracle's elimination-among-winners chain, bit for bit)
  if (upd && sm.Uout && lane < CW - K) {
    double uv = 0.0;
#pragma unroll
    for (int k = K; k < CW; k++) uv = (lane == k - K) ? u[k] : uv;
    const int c = warp_id() + NW * (K + lane);
    if (c > t - 1 && c < sm.ldu) sm.Uout[(int64_t)(t - 1) * sm.ldu + c] = uv;  // single panel: w = n = ldu
  }
  SEL_TRACE(t * 32 + warp_id() * 2 + 1)
}

// Steps t = K*NW + j, j < NW (local pivot column K), then the next group.
template <int W, int NW, int RS, int K>
struct SelGroup {
  static RLHC_DEV void run(double (&a)[RS][W / NW], unsigned& act, int steps, SelSmem<W, NW, RS>& sm) {
    if (K * NW >= steps) return;
    const int q = warp_id();
#pragma unroll 1
    for (int j = 0; j < NW; j++) {
      const int t = K * NW + j;
      if (t < steps) sel_step<W, NW, RS, K>(a, act, t, j == q, sm);
    }
    SelGroup<W, NW, RS, K + 1>::run(a, act, steps, sm);
  }
};
template <int W, int NW, int RS>
struct SelGroup<W, NW, RS, W / NW> {
  static RLHC_DEV void run(double (&)[RS][W / NW], unsigned&, int, SelSmem<W, NW, RS>&) {}
};

// Initialise the step barriers; call before the candidate loads (gepp_select's first
// __syncthreads publishes them).
template <int W, int NW, int RS>
RLHC_DEV void sel_init(SelSmem<W, NW, RS>& sm, double* Uout = nullptr, int ldu = 0) {
  for (int t = threadIdx.x; t < W; t += blockDim.x) mbar_init(&sm.bar[t], 32);
  if (threadIdx.x == 0) {
    sm.Uout = Uout;
    sm.ldu = ldu;
  }
}

template <int W, int NW, int RS>
RLHC_DEV void sel_root_finish(const SelSmem<W, NW, RS>& sm, int steps, int w, const RootOut& ro) {
  if (threadIdx.x == 0 && steps < w) report(ro.status, RLHC_ERANKDEF, RLHC_STAGE_LU, steps);
  for (int t = threadIdx.x; t < steps; t += blockDim.x) {
    ro.piv[t] = sm.out_id[t];
    const int zf = sm.zero[t];
    if (zf == 1) report(ro.status, RLHC_ERANKDEF, RLHC_STAGE_LU, t);
    ro.rdiag[t] = zf == 1 ? 0.0 : (zf < 0 ? -sm.r[t] : sm.r[t]);
  }
  for (int e = threadIdx.x; e < steps * w; e += blockDim.x) {
    const int t = e / w, j = e - t * w;
    double v = 0.0;
    if (j == t) {
      v = 1.0;
    } else if (j < t) {  // l_j of pivot row t: col_j(row) * (1/pivot_j), as every warp formed it
      const int zf = sm.zero[j];
      const double r = zf < 0 ? -sm.r[j] : sm.r[j];
      v = zf == 1 ? 0.0 : __dmul_rn(sm.col[j][sm.out_src[t]], r);
    }
    ro.L11[(int64_t)t * ro.n + j] = v;
  }
}

// GEPP selection (definition: oracle gepp_select / DESIGN.md R#4-R#5).
// a[s][k]: this lane's values (column q + NW k); act: bit s = row (lane + 32 s) is an active
// candidate; gid[s]: global ids, increasing in the candidate index lane + 32 s over the
// active candidates (the tie rule relies on it).  Returns the number of steps; sm.out_id /
// sm.out_src hold the winners (out_src = candidate index lane + 32 s).
template <int W, int NW, int RS>
RLHC_DEV int gepp_select(double (&a)[RS][W / NW], unsigned act, const int (&gid)[RS], int w,
                         SelSmem<W, NW, RS>& sm) {
  if (warp_id() == 0) {
#pragma unroll
    for (int s = 0; s < RS; s++) sm.cgid[s * 32 + lane_id()] = gid[s];
  }
  __syncthreads();  // barrier initialisation visible to every warp
  int c = __popc(act);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  const int steps = min(c, w);
  SelGroup<W, NW, RS, 0>::run(a, act, steps, sm);
  __syncthreads();
  for (int t = threadIdx.x; t < steps; t += blockDim.x) {
    const int src = sm.prow[t];
    sm.out_src[t] = src;
    sm.out_id[t] = sm.cgid[src];
  }
  __syncthreads();
  return steps;
}

}  // namespace rlhc
