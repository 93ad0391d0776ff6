// tslu.cu -- tournament-pivoted tall-skinny LU "PX = LU"
// under the pivot contract of DESIGN.md R#3-R#5 (tslu over column panels).
//
// One select CTA holds up to R = 32*NW candidate rows of a W-wide panel in REGISTERS
// (lane = candidate row, a[W] per lane) and runs GEPP on them: per step one warp
// argmax (redux.sync on the |a| bit pattern, smallest global id on ties), one
// __syncthreads, a cross-warp argmax over NW slots, then a register-resident rank-1
// update whose pivot row comes from shared memory (each warp's local winner writes
// its row speculatively before the barrier, so a step costs one block barrier).
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

template <int W, int NW>
struct SelSmem {
  unsigned long long key[2][NW];
  int id[2][NW];
  double row[2][NW][W];
  int out_src[W];
  int out_id[W];
};

// GEPP selection on the block's candidates (definition: oracle gepp_select / R#4-R#5).
// a: this lane's candidate row (W panel values, entries >= w are ignored), active:
// lane holds a candidate, gid: its global row id, slot: where its original values live.
// Returns the number of steps; sm.out_id[t] / sm.out_src[t] hold the winners.
// The step loop is compile-time recursion (SelStep<.., t>) so every a[] index is a
// constant and the candidate row never leaves the register file.
template <int W, int NW, int t>
struct SelStep {
  static __device__ __forceinline__ void run(double (&a)[W], bool& active, int gid, int slot, int steps,
                                             SelSmem<W, NW>& sm) {
    if (t >= steps) return;
    const int lane = lane_id(), wp = warp_id();
    constexpr int par = t & 1;
    long long kb = active ? __double_as_longlong(fabs(a[t])) : -1ll;
    int hi = (int)(kb >> 32);
    int mh = __reduce_max_sync(0xffffffffu, hi);
    unsigned lo = (hi == mh) ? (unsigned)kb : 0u;
    unsigned ml = __reduce_max_sync(0xffffffffu, lo);
    bool tie = active && hi == mh && (unsigned)kb == ml;
    int wmin = __reduce_min_sync(0xffffffffu, tie ? gid : INT_MAX);
    bool wwin = tie && gid == wmin;
    if (wwin) {
      sm.key[par][wp] = (unsigned long long)kb;
      sm.id[par][wp] = gid;
#pragma unroll
      for (int c = t; c < W; c++) sm.row[par][wp][c] = a[c];
    }
    if (lane == 0 && mh < 0) { sm.key[par][wp] = 0ull; sm.id[par][wp] = INT_MAX; }
    __syncthreads();
    // cross-warp argmax (every warp redundantly)
    unsigned long long k2 = lane < NW ? sm.key[par][lane] : 0ull;
    int id2 = lane < NW ? sm.id[par][lane] : INT_MAX;
    unsigned h2 = (unsigned)(k2 >> 32);
    unsigned gh = __reduce_max_sync(0xffffffffu, h2);
    unsigned l2 = (h2 == gh) ? (unsigned)k2 : 0u;
    unsigned gl = __reduce_max_sync(0xffffffffu, l2);
    bool tie2 = h2 == gh && (unsigned)k2 == gl;
    int pid = __reduce_min_sync(0xffffffffu, tie2 ? id2 : INT_MAX);
    unsigned wmask = __ballot_sync(0xffffffffu, lane < NW && id2 == pid);
    int ww = __ffs(wmask) - 1;
    bool zero = (gh == 0u && gl == 0u);
    if (active && gid == pid) {
      active = false;
      sm.out_src[t] = slot;
    } else if (active && !zero) {
      double u = sm.row[par][ww][t];
      double r = __ddiv_rn(1.0, u);
      double l = __dmul_rn(a[t], r);
#pragma unroll
      for (int c = t + 1; c < W; c++) a[c] = __fma_rn(-l, sm.row[par][ww][c], a[c]);
    }
    if (threadIdx.x == 0) sm.out_id[t] = pid;
    SelStep<W, NW, t + 1>::run(a, active, gid, slot, steps, sm);
  }
};
template <int W, int NW>
struct SelStep<W, NW, W> {
  static __device__ __forceinline__ void run(double (&)[W], bool&, int, int, int, SelSmem<W, NW>&) {}
};

template <int W, int NW>
__device__ __forceinline__ int gepp_select(double (&a)[W], bool active, int gid, int slot, int w,
                                           SelSmem<W, NW>& sm) {
  int nact = __syncthreads_count(active);
  const int steps = min(nact, w);
  SelStep<W, NW, 0>::run(a, active, gid, slot, steps, sm);
  __syncthreads();
  return steps;
}

// Leaf select: leaf = global row block [leaf*R, leaf*R + R) of the LOCAL rows
// (global id = row0 + local row).  src: current values (X for the first panel, the
// trailing matrix afterwards), panel columns [p0, p0 + w).  Output level slot = leaf.
template <int W, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_leaf_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                 const uint8_t* __restrict__ chosen, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals) {
  constexpr int R = 32 * NW;
  __shared__ SelSmem<W, NW> sm;
  const int64_t r = (int64_t)blockIdx.x * R + threadIdx.x;
  bool active = r < rows && !(chosen && chosen[r]);
  double a[W];
  const double* p = src + r * lds + p0;
#pragma unroll
  for (int c = 0; c < W; c++) a[c] = (active && c < w) ? p[c] : 0.0;
  int steps = gepp_select<W, NW>(a, active, (int)(row0 + r), threadIdx.x, w, sm);
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
// child c's k-th winner sits on thread (c - c0)*w + k.  Values are the stored
// current panel values of the candidates (not the eliminated ones).
template <int W, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
tslu_node_kernel(const int* __restrict__ in_ids, const int* __restrict__ in_cnt, const double* __restrict__ in_vals,
                 int nslots_in, int arity, int w, int* __restrict__ out_ids, int* __restrict__ out_cnt,
                 double* __restrict__ out_vals) {
  __shared__ SelSmem<W, NW> sm;
  const int c0 = blockIdx.x * arity;
  const int ci = threadIdx.x / w, e = threadIdx.x - ci * w;
  const int child = c0 + ci;
  bool active = ci < arity && child < nslots_in && e < in_cnt[child < nslots_in ? child : 0];
  const int slot = child * W + e;
  double a[W];
  const double* p = in_vals + (size_t)slot * W;
#pragma unroll
  for (int c = 0; c < W; c++) a[c] = (active && c < w) ? p[c] : 0.0;
  int gid = active ? in_ids[slot] : INT_MAX;
  int steps = gepp_select<W, NW>(a, active, gid, slot, w, sm);
  int* oi = out_ids + (size_t)blockIdx.x * W;
  double* ov = out_vals + (size_t)blockIdx.x * W * W;
  if (threadIdx.x == 0) out_cnt[blockIdx.x] = steps;
  for (int q = threadIdx.x; q < W; q += blockDim.x) oi[q] = q < steps ? sm.out_id[q] : -1;
  for (int idx = threadIdx.x; idx < steps * w; idx += blockDim.x) {
    int q = idx / w, c = idx - q * w;
    ov[q * W + c] = in_vals[(size_t)sm.out_src[q] * W + c];
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
                         unsigned long long* status) {
  __shared__ double P[64][65];
  __shared__ double rd[64];
  __shared__ int ids[64];
  const int tid = threadIdx.x;
  if (tid == 0 && root_cnt[0] < w) report(status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + root_cnt[0]);
  for (int t = tid; t < w; t += blockDim.x) {
    int g = root_ids[t];
    ids[t] = g < 0 ? (int)row0 : g;  // defensive: a short root reports ERANKDEF above
    piv[p0 + t] = g;
    int64_t lr = (int64_t)ids[t] - row0;
    if (chosen && lr >= 0 && lr < rows) chosen[lr] = 1;
  }
  __syncthreads();
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    int t = idx / w, c = idx - t * w;
    P[t][c] = src[((int64_t)ids[t] - row0) * lds + p0 + c];
  }
  __syncthreads();
  // phase A: right-looking elimination of the w x w block (P[t][t'] <- multiplier for t' < t)
  for (int k = 0; k < w; k++) {
    double ukk = P[k][k];
    if (tid == 0) {
      if (ukk == 0.0) report(status, RLHC_ERANKDEF, RLHC_STAGE_LU, p0 + k);
      rd[k] = __ddiv_rn(1.0, ukk);
    }
    __syncthreads();
    double r = rd[k];
    int cnt = (w - 1 - k) * (w - k);  // rows k+1..w-1, columns k..w-1 (col k = multiplier)
    for (int idx = tid; idx < (w - 1 - k); idx += blockDim.x) {
      int t = k + 1 + idx;
      P[t][k] = __dmul_rn(P[t][k], r);
    }
    __syncthreads();
    (void)cnt;
    for (int idx = tid; idx < (w - 1 - k) * (w - 1 - k); idx += blockDim.x) {
      int t = k + 1 + idx / (w - 1 - k), c = k + 1 + idx % (w - 1 - k);
      P[t][c] = __fma_rn(-P[t][k], P[k][c], P[t][c]);
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
        double v = src[((int64_t)ids[t] - row0) * lds + j];
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

template <int W, int NW>
static cudaError_t run_leaf(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                            const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st) {
  int nleaves = (int)ceil_div<int64_t>(rows, 32 * NW);
  tslu_leaf_kernel<W, NW><<<nleaves, 32 * NW, 0, st>>>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals);
  return cudaGetLastError();
}
template <int W, int NW>
static cudaError_t run_node(const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity, int w,
                            int* ids, int* cnt, double* vals, cudaStream_t st) {
  int nout = ceil_div(nin, arity);
  tslu_node_kernel<W, NW><<<nout, 32 * NW, 0, st>>>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals);
  return cudaGetLastError();
}

cudaError_t launch_tslu_leaf(int W, const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                             const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st) {
  switch (W) {
    case 16: return run_leaf<16, 16>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st);
    case 32: return run_leaf<32, 16>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st);
    case 64: return run_leaf<64, 8>(src, lds, rows, row0, p0, w, chosen, ids, cnt, vals, st);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_tslu_node(int W, const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity,
                             int w, int* ids, int* cnt, double* vals, cudaStream_t st) {
  switch (W) {
    case 16: return run_node<16, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st);
    case 32: return run_node<32, 16>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st);
    case 64: return run_node<64, 8>(in_ids, in_cnt, in_vals, nin, arity, w, ids, cnt, vals, st);
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_tslu_panel_factor(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w, int n,
                                     const int* root_ids, const int* root_cnt, double* U, int64_t* piv,
                                     uint8_t* chosen, double* lpanel, unsigned long long* status, cudaStream_t st) {
  tslu_panel_factor_kernel<<<1, 512, 0, st>>>(src, lds, rows, row0, p0, w, n, root_ids, root_cnt, U, piv, chosen,
                                              lpanel, status);
  return cudaGetLastError();
}
cudaError_t launch_l11_fixup(double* L11, int n, cudaStream_t st) {
  l11_fixup_kernel<<<n, 128, 0, st>>>(L11, n);
  return cudaGetLastError();
}
cudaError_t launch_gather_rows(const double* src, int64_t lds, const int64_t* ids, int64_t row0, int cnt, int ncols,
                               double* dst, int64_t ldd, cudaStream_t st) {
  gather_rows_kernel<<<cnt, 128, 0, st>>>(src, lds, ids, row0, cnt, ncols, dst, ldd);
  return cudaGetLastError();
}
cudaError_t launch_pivpos(const int64_t* piv, int n, int64_t row0, int64_t rows, int* pivpos, cudaStream_t st) {
  pivpos_kernel<<<ceil_div(n, 128), 128, 0, st>>>(piv, n, row0, rows, pivpos);
  return cudaGetLastError();
}

}  // namespace rlhc
