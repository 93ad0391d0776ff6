// select.cuh -- the GEPP "select" of one tournament node (R#4-R#5), used by the
// leaf and node kernels of tslu.cu.
//
// Column-owned layout: CTA = NW warps, R = 32*RS candidate rows, panel width W; warp q
// owns the CW = W/NW panel columns [q*CW, q*CW+CW) of ALL R rows, lane l holds rows
// {l + 32 s : s < RS}, so a[s][c] = row (l + 32 s), column q*CW + c.
//
// Step t (pivot column t, owned by warp q = t / CW at local column CC):
//   * after the barrier that published step t-1 (multipliers l, pivot row index), the
//     owner warp first applies step t-1's update to column CC only, takes the warp-local
//     argmax of |a[.][CC]| (ties -> smallest global id; no cross-warp reduction), forms
//     the multipliers a_rt / a_pt and publishes them through shared memory, and only
//     then applies step t-1's update to its other columns;
//   * every other warp applies step t-1's update to its columns (the pivot row's values
//     come from its own registers: select + shuffle from the owning lane);
//   * ONE __syncthreads per step.
// The per-element fma chain (increasing step order) is unchanged, so the pivots are
// bit-identical to the oracle's gepp_select.
#pragma once
#include <climits>

#include "common.cuh"

namespace rlhc {

template <int W, int NW, int RS>
struct SelSmem {
  double l[2][32 * RS];
  int prow[2];  // candidate index of the pivot row
  int zero[2];  // zero pivot column (R#5: no update)
  int out_src[W];
  int out_id[W];
};

// v[c - C_LO] = a[pslot][c] for a warp-uniform runtime slot (compile-time recursion over
// slots -> a chain of uniform branches, each copying statically indexed registers)
template <int W, int NW, int RS, int C_LO, int C_HI, int S>
__device__ __forceinline__ void sel_extract(const double (&a)[RS][W / NW], int pslot, double* v) {
  if constexpr (S < RS) {
    if (pslot == S) {
#pragma unroll
      for (int c = C_LO; c < C_HI; c++) v[c - C_LO] = a[S][c];
    } else {
      sel_extract<W, NW, RS, C_LO, C_HI, S + 1>(a, pslot, v);
    }
  }
}

// Apply the published step (par) to columns [c_lo, c_hi) of this warp (compile-time
// bounds), for the rows still active after removing the pivot row.
template <int W, int NW, int RS, int C_LO, int C_HI>
__device__ __forceinline__ void sel_apply(double (&a)[RS][W / NW], unsigned act, int pslot, int plane, int par,
                                          const SelSmem<W, NW, RS>& sm) {
  if (C_LO >= C_HI) return;
  __syncwarp();
  double u[C_HI > C_LO ? C_HI - C_LO : 1];
#pragma unroll
  for (int c = C_LO; c < C_HI; c++) {
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < RS; s++) v = (s == pslot) ? a[s][c] : v;
    u[c - C_LO] = __shfl_sync(0xffffffffu, v, plane);
  }
  // applied to every slot without a branch (keeps the warp converged for the collectives
  // that follow): rows no longer in the candidate set are never read again
#pragma unroll
  for (int s = 0; s < RS; s++) {
    const double l = sm.l[par][s * 32 + lane_id()];
#pragma unroll
    for (int c = C_LO; c < C_HI; c++) a[s][c] = __fma_rn(-l, u[c - C_LO], a[s][c]);
  }
  (void)act;
}

// Argmax + publish for pivot column CC of the calling (owner) warp, step t.
template <int W, int NW, int RS, int CC>
__device__ __forceinline__ void sel_pivot(double (&a)[RS][W / NW], unsigned act, const int (&gid)[RS], int t,
                                          SelSmem<W, NW, RS>& sm) {
  const int lane = lane_id();
  const int par = t & 1;
  __syncwarp();
  long long bk = -1ll;
  int bid = INT_MAX, bs = 0;
#pragma unroll
  for (int s = 0; s < RS; s++) {
    long long k = ((act >> s) & 1u) ? __double_as_longlong(fabs(a[s][CC])) : -1ll;
    bool better = k > bk || (k == bk && gid[s] < bid);
    bk = better ? k : bk; bid = better ? gid[s] : bid; bs = better ? s : bs;
  }
  int hi = (int)(bk >> 32);
  int mh = __reduce_max_sync(0xffffffffu, hi);
  unsigned lo = (hi == mh) ? (unsigned)bk : 0u;
  unsigned ml = __reduce_max_sync(0xffffffffu, lo);
  bool tie = bk >= 0 && hi == mh && (unsigned)bk == ml;
  int pid = __reduce_min_sync(0xffffffffu, tie ? bid : INT_MAX);
  const unsigned wm = __ballot_sync(0xffffffffu, tie && bid == pid);
  const int plane = __ffs(wm) - 1;
  double mv = 0.0;
#pragma unroll
  for (int s = 0; s < RS; s++) mv = (s == bs) ? a[s][CC] : mv;
  const double pv = __shfl_sync(0xffffffffu, mv, plane);
  const int pslot = __shfl_sync(0xffffffffu, bs, plane);
  const bool zero = (mh == 0 && ml == 0u);
  const double r = zero ? 0.0 : __drcp_rn(pv);  // correctly rounded 1/pv (== IEEE 1.0/pv)
#pragma unroll
  for (int s = 0; s < RS; s++) sm.l[par][s * 32 + lane] = zero ? 0.0 : __dmul_rn(a[s][CC], r);
  if (lane == 0) {
    sm.prow[par] = pslot * 32 + plane;
    sm.zero[par] = zero;
    sm.out_src[t] = pslot * 32 + plane;
    sm.out_id[t] = pid;
  }
}

// Step t with pivot column (warp q, local column CC): finish step t-1 (delayed update),
// pivot search for step t, barrier.
template <int W, int NW, int RS, int CC>
__device__ __forceinline__ void sel_step(double (&a)[RS][W / NW], unsigned& act, const int (&gid)[RS], int t, int q,
                                         SelSmem<W, NW, RS>& sm) {
  constexpr int CW = W / NW;
  const int wp = warp_id();
  bool prev = false;
  int pslot = 0, plane = 0, ppar = (t - 1) & 1;
  if (t > 0) {
    const int prow = sm.prow[ppar];
    pslot = prow >> 5; plane = prow & 31;
    if (lane_id() == plane) act &= ~(1u << pslot);  // the pivot row of step t-1 leaves the set
    prev = !sm.zero[ppar];
  }
  if (wp == q) {
    // the previous step's update of the pivot column first, then the argmax
    if (prev) sel_apply<W, NW, RS, CC, CC + 1>(a, act, pslot, plane, ppar, sm);
    sel_pivot<W, NW, RS, CC>(a, act, gid, t, sm);
    if (prev) sel_apply<W, NW, RS, CC + 1, CW>(a, act, pslot, plane, ppar, sm);
  } else if (prev && wp > q) {
    sel_apply<W, NW, RS, 0, CW>(a, act, pslot, plane, ppar, sm);
  }
  __syncthreads();
}

template <int W, int NW, int RS, int CC>
struct SelGroup {
  static __device__ __forceinline__ void run(double (&a)[RS][W / NW], unsigned& act, const int (&gid)[RS], int t0,
                                             int steps, int q, SelSmem<W, NW, RS>& sm) {
    if (t0 + CC >= steps) return;
    sel_step<W, NW, RS, CC>(a, act, gid, t0 + CC, q, sm);
    SelGroup<W, NW, RS, CC + 1>::run(a, act, gid, t0, steps, q, sm);
  }
};
template <int W, int NW, int RS>
struct SelGroup<W, NW, RS, W / NW> {
  static __device__ __forceinline__ void run(double (&)[RS][W / NW], unsigned&, const int (&)[RS], int, int, int,
                                             SelSmem<W, NW, RS>&) {}
};

// GEPP selection (definition: oracle gepp_select / DESIGN.md R#4-R#5).
// a[s][c]: this lane's values; act: bit s = row (lane + 32 s) is an active candidate;
// gid[s]: global ids.  Returns the number of steps; sm.out_id / sm.out_src hold the
// winners (out_src = candidate index lane + 32 s).
template <int W, int NW, int RS>
__device__ __forceinline__ int gepp_select(double (&a)[RS][W / NW], unsigned act, const int (&gid)[RS], int w,
                                           SelSmem<W, NW, RS>& sm) {
  constexpr int CW = W / NW;
  int c = __popc(act);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  const int steps = min(c, w);
#pragma unroll 1
  for (int q = 0; q * CW < steps; q++) SelGroup<W, NW, RS, 0>::run(a, act, gid, q * CW, steps, q, sm);
  __syncthreads();
  return steps;
}

}  // namespace rlhc
