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

}  // namespace

bool subst_wide_ok(int n) { return n > 64 && sw_smem_bytes(n) <= 227 * 1024; }

// out = A T^{-1} in the oracle's operation order (n > 64).  out may be A itself (block b reads
// its inputs before writing them and re-reads only the earlier blocks' outputs), not a partial
// overlap.  T's diagonal is checked separately (launch_rdiag).
cudaError_t launch_subst_wide(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                              double* out, int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
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
