// subst.cu -- W = X Y^-1 ("Q = X R^{-1}" of SLHC) by row substitution in the oracle's
// operation order (DESIGN.md R#O9, ora_trsm_right_upper) for n > 64:
//   acc = x_k;  acc = RN(acc - RN(w_j Y_jk)) for j = 0 .. k-1 (increasing);  w_k = RN(acc / Y_kk)
// so W is bit-identical to the oracle's at every n.  No fused multiply-add: each term costs a
// DMUL and a DADD, twice the FP64 issue of the fma chain -- the price of this order, which
// keeps the arrowhead family of P:1071-1082 from breaking down (R#O9).
//
// Thread = row (128 rows per CTA, several CTAs per SM), 32-column blocks.  For block b the
// thread's 32 accumulators (registers) start from x and receive, LEFT-looking, the terms of
// the earlier outputs j < 32 b in increasing j: chunk by chunk the CTA stages its rows'
// outputs of an earlier block jc (written to `out` before; 128 x 32 doubles from L2) and
// Y[32 jc .. +32][32 b .. +32] in shared memory (Y rows are broadcast reads).  Then the
// block's own columns are solved RIGHT-looking in registers with static indices (rotated: at
// step k acc[0] is column 32 b + k), each output divided exactly (div_by_rcp == IEEE
// division) and the later columns receiving RN(acc - RN(w_k Y_kc)).  Per element: the
// oracle's terms, order and roundings.  (A first version with 8 threads per row and the
// in-block chain passed by shuffles ran at 41 % of the FP64 pipe: 3.5x the instructions.)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {
namespace {

constexpr int SW_R = 128;                    // rows (threads) per CTA
constexpr int SW_B = 32;                     // column block
constexpr int SW_LD = SW_B + 1;              // staged row stride (doubles): conflict-free per-thread rows

__host__ __device__ inline size_t sw_smem_bytes(int n) {
  return ((size_t)SW_R * SW_LD + (size_t)SW_B * SW_B + 2 * (size_t)n) * sizeof(double);
}

// a / b correctly rounded from y = RN(1/b) (rows.cu's div_by_rcp)
__device__ __forceinline__ double sw_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q1 = __fma_rn(__fma_rn(-b, q0, a), y, q0);
  const double q2 = __fma_rn(__fma_rn(-b, q1, a), y, q1);
  const double aa = fabs(a), aq = fabs(q2);
  if (aa >= 0x1p-900 && aa <= 0x1p+900 && aq >= 0x1p-900 && aq <= 0x1p+900) return q2;
  return __ddiv_rn(a, b);
}

__global__ void __launch_bounds__(SW_R, 4)
subst_wide_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int n, const double* __restrict__ T,
                  int64_t ldt, double* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) double sw_sm[];
  double* St = sw_sm;                    // [SW_R][SW_LD]: x of block b, the outputs of block jc, staging
  double* Tb = St + SW_R * SW_LD;        // [SW_B][SW_B]
  double* dg = Tb + SW_B * SW_B;         // [n] Y_kk, [n] RN(1/Y_kk)
  const int tid = threadIdx.x;
  const int nb = ceil_div(n, SW_B);
  pdl_trigger();
  pdl_wait();
  for (int k = tid; k < n; k += SW_R) {
    const double d = T[(int64_t)k * ldt + k];
    const double ad = fabs(d);
    dg[k] = d;
    dg[n + k] = (ad >= 0x1p-900 && ad <= 0x1p+900) ? __drcp_rn(d) : __longlong_as_double(0x7ff8000000000000LL);
  }
  // St <- src[r0 .. r0 + 128][cs .. cs + 32];  Tb <- Y[j0 .. j0 + 32][c0 .. c0 + 32]
  // thread tid copies column c = tid & 31 of rows q = (tid >> 5) + 4 i (one 8-byte copy each;
  // 32 consecutive threads cover 256 contiguous bytes of a row)
  const int cq = tid >> 5, cc = tid & 31;
  auto stage = [&](const double* src, int64_t lds, int64_t r0, int cs, int j0, int c0) {
    __syncthreads();  // St / Tb free
    if (src) {
      const bool cin = cs + cc < n;
      const double* s0 = src + (r0 + cq) * lds + cs + cc;
      double* d0 = St + cq * SW_LD + cc;
      const int64_t step = 4 * lds;
#pragma unroll
      for (int i = 0; i < SW_R / 4; i++) {
        const bool in = cin && r0 + cq + 4 * i < rows;
        cp_async8(d0 + 4 * i * SW_LD, in ? s0 + i * step : src, in ? 8 : 0);
      }
    }
    {
      const bool cin = c0 + cc < n;
      const double* s0 = T + (int64_t)(j0 + cq) * ldt + c0 + cc;
#pragma unroll
      for (int i = 0; i < SW_B / 4; i++) {
        const bool in = cin && j0 + cq + 4 * i < n;
        cp_async8(Tb + (cq + 4 * i) * SW_B + cc, in ? s0 + (int64_t)4 * i * ldt : T, in ? 8 : 0);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  };
  const double* st_row = St + tid * SW_LD;
  const int64_t ntiles = ceil_div<int64_t>(rows, SW_R);
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t r0 = tl * SW_R;
    for (int b = 0; b < nb; b++) {
      const int c0 = b * SW_B;
      double acc[SW_B];
      stage(A, lda, r0, c0, 0, c0);  // x of block b (Tb: Y[0..32][block b], the first chunk's)
#pragma unroll
      for (int c = 0; c < SW_B; c++) acc[c] = st_row[c];
      for (int jc = 0; jc < b; jc++) {
        // terms of the outputs of block jc, j increasing
        stage(out, ldo, r0, jc * SW_B, jc * SW_B, c0);
#pragma unroll 2
        for (int jj = 0; jj < SW_B; jj++) {
          const double w = st_row[jj];
          const double* y = Tb + jj * SW_B;
#pragma unroll
          for (int c = 0; c < SW_B; c += 2) {
            const double2 yy = *reinterpret_cast<const double2*>(y + c);
            acc[c] = __dsub_rn(acc[c], __dmul_rn(w, yy.x));
            acc[c + 1] = __dsub_rn(acc[c + 1], __dmul_rn(w, yy.y));
          }
        }
      }
      if (b > 0) stage(nullptr, 0, r0, 0, c0, c0);  // the diagonal block of Y
      // right-looking in registers, rotated: at step k acc[0] is column c0 + k; each output goes
      // straight to the thread's own staging row (St's staged values are no longer needed)
      double* wr = St + tid * SW_LD;
#pragma unroll
      for (int k = 0; k < SW_B; k++) {
        const int kk = c0 + k;
        const double w = kk < n ? sw_div(acc[0], dg[kk], dg[n + kk]) : 0.0;
        wr[k] = w;
        const double* y = Tb + k * SW_B + k;  // y[c] = Y[kk][kk + c]
#pragma unroll
        for (int c = 1; c < SW_B - k; c++) acc[c - 1] = __dsub_rn(acc[c], __dmul_rn(w, y[c]));
      }
      // outputs of block b -> out, staged for coalesced stores
      __syncthreads();
      if (c0 + cc < n) {
        double* o0 = out + (r0 + cq) * ldo + c0 + cc;
#pragma unroll 8
        for (int i = 0; i < SW_R / 4; i++)
          if (r0 + cq + 4 * i < rows) o0[(int64_t)4 * i * ldo] = St[(cq + 4 * i) * SW_LD + cc];
      }
    }
  }
}


// ---------------------------------------------------------------- TMA variant (default)
// The same per-element arithmetic, restructured so that the FP64 pipe, not the load path,
// sets the pace.  A DMUL or a DADD occupies the FP64 pipe as long as a DFMA (16 lanes per
// clock per SMSP; tools/probe/pdmuladd.cu: a DMUL + DADD term runs at half the DFMA term
// rate, and DMMA shares the same units, tools/probe/pmix.cu), so the kernel's roof is one
// term per 2 pipe slots, and the loads and address arithmetic must hide in the issue slots
// the FP64 pipe leaves free:
//  * each consumer thread owns TWO rows (t and t + SV_T of the tile) and a 16-column block:
//    every Y element loaded (a warp-uniform broadcast) serves two terms, and one 16-byte load
//    per row brings the w of two j -- 9 loads per 64 FP64 instructions;
//  * a warp-specialised producer thread streams items into SV_NS shared-memory slots with 2-D
//    TMA copies completing on the slot's `full` mbarrier: per 16-column block b, X (the tile's
//    x), then for jc < b the outputs of block jc (re-read from `out`; 128B swizzle, so the
//    thread = row 16-byte reads are conflict-free) with Y[16 jc .. +16][16 b .. +16]
//    (unswizzled: broadcast reads), then D (Y's diagonal block);
//  * the outputs of block b are written into D's row box and leave by TMA store, issued by
//    the producer (after the consumers' fence.proxy.async + empty arrival) when it next
//    reuses that slot or, earlier, before it loads that block back from `out` -- so no
//    consumer waits on a store, and every re-read follows its store's completion.
constexpr int SV_CW = 4;                      // consumer warps per CTA
constexpr int SV_T = 32 * SV_CW;              // consumer threads; rows t and t + SV_T
constexpr int SV_R = 2 * SV_T;                // rows per tile
constexpr int SV_B = 16;                      // column block (= one 128-byte row box)
constexpr int SV_NS = 3;                      // slots
constexpr int SV_THREADS = SV_T + 32;
struct __align__(1024) SvSlot {
  double O[SV_R][SV_B];                       // one row box, 128B-swizzled
  double Y[SV_B][SV_B];                       // 16 x 16 of Y, unswizzled
};
struct __align__(1024) SvSmem {
  SvSlot slot[SV_NS];
  unsigned long long full[SV_NS], empty[SV_NS];
};
__device__ __forceinline__ void sv_tma_load(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sv_tma_store(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void sv_tma_load_h(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void sv_tma_store_h(const CUtensorMap* map, int x, int y, const void* src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void sv_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// (row r, column c < 16) of a swizzled row box, in doubles
__device__ __forceinline__ int sv_off(int r, int c) { return r * SV_B + ((((c >> 1) ^ r) & 7) << 1) + (c & 1); }

__global__ void __launch_bounds__(SV_THREADS, 2)
subst_wide_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmO,
                      const __grid_constant__ CUtensorMap tmT, int64_t rows, int n, const double* __restrict__ T,
                      int64_t ldt, int hint) {
  extern __shared__ __align__(1024) unsigned char sv_raw[];
  SvSmem& sm = *reinterpret_cast<SvSmem*>(sv_raw + ((1024u - (smem_u32(sv_raw) & 1023u)) & 1023u));
  double* dg = reinterpret_cast<double*>(&sm + 1);  // [n] Y_kk, [n] RN(1/Y_kk)
  const int tid = threadIdx.x, lane = lane_id(), wp = warp_id();
  const int nb = ceil_div(n, SV_B);
  const int64_t ntiles = ceil_div<int64_t>(rows, SV_R);
  if (tid < SV_NS) {
    mbar_init(&sm.full[tid], 1);
    mbar_init(&sm.empty[tid], SV_CW);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  pdl_trigger();
  pdl_wait();
  for (int k = tid; k < n; k += SV_THREADS) {
    const double d = T[(int64_t)k * ldt + k];
    const double ad = fabs(d);
    dg[k] = d;
    dg[n + k] = (ad >= 0x1p-900 && ad <= 0x1p+900) ? __drcp_rn(d) : __longlong_as_double(0x7ff8000000000000LL);
  }
  __syncthreads();
  if (wp == SV_CW) {
    // ---------------- producer (one thread)
    if (lane != 0) return;
    // hint (measurement knob RLHC_SV_HINT): X is read once (evict first), the outputs are
    // re-read by the tile's later blocks (evict last)
    uint64_t pol_first = 0, pol_last = 0;
    if (hint) {
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_last));
    }
    int pend_b[SV_NS], pend_r0[SV_NS];  // a D item's output box still to be stored from the slot
    uint32_t pend_q[SV_NS];
    for (int s = 0; s < SV_NS; s++) pend_b[s] = -1, pend_r0[s] = 0, pend_q[s] = 0;
    uint32_t q = 0;
    // store slot s's pending output box (waiting for the consumers to release it first)
    auto flush = [&](int s) {
      if (pend_b[s] < 0) return;
      mbar_wait(&sm.empty[s], (pend_q[s] / SV_NS) & 1);  // D's consumers are done with the slot
      if (hint) sv_tma_store_h(&tmO, pend_b[s] * SV_B, pend_r0[s], &sm.slot[s].O[0][0], pol_last);
      else sv_tma_store(&tmO, pend_b[s] * SV_B, pend_r0[s], &sm.slot[s].O[0][0]);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      pend_b[s] = -1;
    };
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      const int r0 = (int)(tl * SV_R);
      for (int b = 0; b < nb; b++) {
        for (int e = -1; e <= b; e++, q++) {  // -1: X;  0 .. b-1: outputs of block e;  b: D
          const int s = q % SV_NS;
          if (q >= SV_NS) {
            if (pend_b[s] >= 0) flush(s);     // waits for the slot's release itself
            else mbar_wait(&sm.empty[s], ((q / SV_NS) - 1) & 1);
          }
          SvSlot& sl = sm.slot[s];
          if (e < 0) {
            sv_expect_tx(&sm.full[s], SV_R * SV_B * 8u);
            if (hint) sv_tma_load_h(&sl.O[0][0], &tmA, b * SV_B, r0, &sm.full[s], pol_first);
            else sv_tma_load(&sl.O[0][0], &tmA, b * SV_B, r0, &sm.full[s]);
          } else if (e < b) {
            for (int k = 0; k < SV_NS; k++)   // block e's outputs must be in `out` first
              if (pend_b[k] == e && pend_r0[k] == r0) flush(k);
            sv_expect_tx(&sm.full[s], SV_R * SV_B * 8u + SV_B * SV_B * 8u);
            if (hint) sv_tma_load_h(&sl.O[0][0], &tmO, e * SV_B, r0, &sm.full[s], pol_last);
            else sv_tma_load(&sl.O[0][0], &tmO, e * SV_B, r0, &sm.full[s]);
            sv_tma_load(&sl.Y[0][0], &tmT, b * SV_B, e * SV_B, &sm.full[s]);
          } else {
            sv_expect_tx(&sm.full[s], SV_B * SV_B * 8u);
            sv_tma_load(&sl.Y[0][0], &tmT, b * SV_B, b * SV_B, &sm.full[s]);
            pend_b[s] = b, pend_r0[s] = r0, pend_q[s] = q;
          }
        }
      }
    }
    for (int s = 0; s < SV_NS; s++) flush(s);
    return;
  }
  // ---------------- consumers: rows t and t + SV_T of the tile
  const int t = tid, sw = t & 7;
  uint32_t q = 0;
  auto take = [&]() -> SvSlot& {
    const int s = q % SV_NS;
    mbar_wait(&sm.full[s], (q / SV_NS) & 1);
    return sm.slot[s];
  };
  auto give = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[q % SV_NS]);
    q++;
  };
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    for (int b = 0; b < nb; b++) {
      const int c0 = b * SV_B;
      double a0[SV_B], a1[SV_B];
      {
        const double* O = &take().O[0][0];
#pragma unroll
        for (int c = 0; c < SV_B; c += 2) {
          const double2 v0 = *reinterpret_cast<const double2*>(O + sv_off(t, c));
          const double2 v1 = *reinterpret_cast<const double2*>(O + sv_off(t + SV_T, c));
          a0[c] = v0.x, a0[c + 1] = v0.y, a1[c] = v1.x, a1[c + 1] = v1.y;
        }
        give();
      }
      for (int e = 0; e < b; e++) {
        SvSlot& sl = take();
        const double* o0 = &sl.O[t][0];
        const double* o1 = &sl.O[t + SV_T][0];
#pragma unroll 2
        for (int jj = 0; jj < SV_B; jj += 2) {
          const int co = (((jj >> 1) ^ sw) & 7) << 1;
          const double2 w0 = *reinterpret_cast<const double2*>(o0 + co);
          const double2 w1 = *reinterpret_cast<const double2*>(o1 + co);
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const double x0 = u ? w0.y : w0.x, x1 = u ? w1.y : w1.x;
            const double* y = &sl.Y[jj + u][0];
#pragma unroll
            for (int c = 0; c < SV_B; c += 2) {
              const double2 yy = *reinterpret_cast<const double2*>(y + c);
              a0[c] = __dsub_rn(a0[c], __dmul_rn(x0, yy.x));
              a0[c + 1] = __dsub_rn(a0[c + 1], __dmul_rn(x0, yy.y));
              a1[c] = __dsub_rn(a1[c], __dmul_rn(x1, yy.x));
              a1[c + 1] = __dsub_rn(a1[c + 1], __dmul_rn(x1, yy.y));
            }
          }
        }
        give();
      }
      // the diagonal block, right-looking in registers (rotated: at step k a[0] is column c0 + k);
      // the outputs go to D's row box, stored by the producer
      {
        SvSlot& sl = take();
        double* wr = &sl.O[0][0];
#pragma unroll
        for (int k = 0; k < SV_B; k++) {
          const int kk = c0 + k < n ? c0 + k : 0;
          const bool in = c0 + k < n;
          const double d = dg[kk], rd = dg[n + kk];
          const double w0 = in ? sw_div(a0[0], d, rd) : 0.0;
          const double w1 = in ? sw_div(a1[0], d, rd) : 0.0;
          wr[sv_off(t, k)] = w0;
          wr[sv_off(t + SV_T, k)] = w1;
          const double* y = &sl.Y[k][0];
#pragma unroll
          for (int c = 1; c < SV_B; c++)
            if (c < SV_B - k) {
              const double yv = y[k + c];
              a0[c - 1] = __dsub_rn(a0[c], __dmul_rn(w0, yv));
              a1[c - 1] = __dsub_rn(a1[c], __dmul_rn(w1, yv));
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        give();
      }
    }
  }
}

}  // namespace

bool subst_wide_ok(int n) { return n > 64 && sw_smem_bytes(n) <= 227 * 1024; }

// out = A T^{-1} in the oracle's operation order (n > 64).  out may be A itself (block b reads
// its inputs before writing them and re-reads only the earlier blocks' outputs), not a partial
// overlap.  T's diagonal is checked separately (launch_rdiag).
static cudaError_t launch_subst_wide_tma(const double* A, int64_t lda, int64_t rows, int n, const double* T,
                                         int64_t ldt, double* out, int64_t ldo, cudaStream_t st, bool* done) {
  *done = false;
  static const bool on = [] { const char* e = getenv("RLHC_SUBST_TMA"); return !e || atoi(e) != 0; }();
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  const bool ok = on && enc && lda % 2 == 0 && ldo % 2 == 0 && ldt % 2 == 0 &&
                  (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(T) & 15) == 0 && rows < (int64_t(1) << 31);
  if (!ok) return cudaSuccess;
  CUtensorMap mA, mO, mT;
  auto make = [&](CUtensorMap* m, const double* base, int64_t ld, int64_t nrows, uint32_t box_cols, uint32_t box_rows,
                  CUtensorMapSwizzle swz) {
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!make(&mA, A, lda, rows, SV_B, SV_R, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make(&mO, out, ldo, rows, SV_B, SV_R, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make(&mT, T, ldt, n, SV_B, SV_B, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaSuccess;
  const int smem = (int)(sizeof(SvSmem) + 2 * (size_t)n * sizeof(double) + 1024);
  if (smem > 227 * 1024) return cudaSuccess;
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, subst_wide_tma_kernel, 227 * 1024)) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) return e;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, subst_wide_tma_kernel, SV_THREADS, smem))
    return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, SV_R),
                                                              (int64_t)sms * std::max(per_sm, 1)));
  note_launch();
  *done = true;
  static const int hint = [] { const char* e = getenv("RLHC_SV_HINT"); return e ? atoi(e) : 1; }();
  return launch_pdl(subst_wide_tma_kernel, dim3((unsigned)grid), dim3(SV_THREADS), (size_t)smem, st, mA, mO, mT, rows,
                    n, T, ldt, hint);
}

cudaError_t launch_subst_wide(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                              double* out, int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  bool done = false;
  if (cudaError_t e = launch_subst_wide_tma(A, lda, rows, n, T, ldt, out, ldo, st, &done)) return e;
  if (done) return cudaSuccess;
  const int smem = (int)sw_smem_bytes(n);
  static DevFlags attr;  // the attribute is the largest size any n may need (set once per device)
  if (cudaError_t e = smem_attr(attr, subst_wide_kernel, 227 * 1024)) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) return e;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, subst_wide_kernel, SW_R, smem))
    return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, SW_R),
                                                              (int64_t)sms * std::max(per_sm, 1)));
  note_launch();
  return launch_pdl(subst_wide_kernel, dim3((unsigned)grid), dim3(SW_R), (size_t)smem, st, A, lda, rows, n, T, ldt,
                    out, ldo);
}

}  // namespace rlhc
