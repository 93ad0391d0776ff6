// syrk.cu -- G = A^T A (the Gram of CholeskyQR) for n <= 256 as a fragment-balanced,
// TMA-fed DMMA pipeline.
//
// The upper triangle of G in 8 x 8 DMMA fragments has NR (NR + 1) / 2 of them (NR = n / 8,
// rounded up to 8, 16 or 32).  Fragment row r holds NR - r of them, so rows r and NR - 1 - r
// together hold NR + 1: warp w owns fragment rows w and NR - 1 - w (w < NR / 2) -- every warp
// has the same work and every fragment of the triangle is computed once (the 64 x 64 tiling of
// gram_kernel left diagonal tiles with one idle and two part-idle warps).  NR / 2 warps in all,
// 8 per CTA (NR = 32: two CTA types, each a persistent CTA per SM streaming every row of A).
// Per CTA, one producer thread moves 32-row chunks of A (every column: 16-column boxes,
// 128-byte swizzle) into S stages by TMA (cp.async.bulk.tensor, completing on the stage's
// `full` mbarrier); the consumer warps wait on `full`, contract, and release `empty` -- no
// CTA barrier.  Lane t of a DMMA k-step reads chunk row 2 t + par (par = 0, 1), so the four
// k rows of a step fall on different 16-byte swizzle phases and every fragment load is
// bank-conflict free.  The warp's fragment rows are template parameters (a switch over the
// warp index), so every fragment address is a per-lane base plus an immediate.
// Each warp's NR + 1 accumulators go to a per-CTA partial; syrk_reduce_kernel sums the
// partials of a fragment's CTA type in increasing CTA order and mirrors -- deterministic, no
// atomics.  The order of the additions differs from gram_kernel's (tolerance-compared like it).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {
namespace {

constexpr int SY_R = 32;         // rows per stage
constexpr int kSyMaxGrid = 296;  // CTAs (the partials are sized for it; a B200 runs 148 or 296)

template <int NR>
struct SyCfg {
  static constexpr int NW = NR / 2;                  // warps over all CTA types
  static constexpr int CW = NW < 8 ? NW : 8;         // consumer warps per CTA
  static constexpr int T = NW / CW;                  // CTA types
  static constexpr int NB = NR / 2;                  // 16-column boxes per row chunk
  static constexpr int F = NR + 1;                   // fragments per warp
  static constexpr uint32_t STAGE = NB * SY_R * 128;  // bytes per stage
  static constexpr int S = (196 * 1024) / STAGE > 6 ? 6 : (196 * 1024) / STAGE;
  static constexpr int THREADS = 32 * (CW + 1);
  static constexpr size_t SMEM = (size_t)S * STAGE + 2 * S * 8 + 1024;
  static constexpr size_t PART = (size_t)CW * F * 64;  // doubles per CTA
};

__device__ __forceinline__ void sy_tma(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sy_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// the consumer loop of warp W (fragment rows W and NR - 1 - W); out: [F][64] of this warp
template <int NR, int W>
__device__ __forceinline__ void sy_consume(const double* stg, unsigned long long* full, unsigned long long* empty,
                                           int64_t nchunks, int64_t cta, int64_t nct, double* __restrict__ out) {
  using C = SyCfg<NR>;
  constexpr int RA = W, RB = NR - 1 - W;
  const int lane = lane_id(), g = lane >> 2, t = lane & 3;
  double acc[C::F][2];
#pragma unroll
  for (int f = 0; f < C::F; f++) acc[f][0] = acc[f][1] = 0.0;
  uint32_t q = 0;
  for (int64_t ch = cta; ch < nchunks; ch += nct, q++) {
    const int s = (int)(q % C::S);
    mbar_wait(&full[s], (q / C::S) & 1);
    const double* st = stg + (size_t)s * (C::STAGE / 8);
#pragma unroll 1
    for (int kb = 0; kb < SY_R / 8; kb++) {
#pragma unroll
      for (int par = 0; par < 2; par++) {
        // column 8 c + g of chunk row kb*8 + 2t + par: box c/2, 16-byte chunk 4 (c%2) + g/2
        // XOR the row's swizzle phase, element g%2
        const int rsw = (2 * t + par) & 7;
        const double* rowp = st + (kb * 8 + 2 * t + par) * 16 + (g & 1);
        const double* p0 = rowp + ((((g >> 1)) ^ rsw) << 1);
        const double* p1 = rowp + (((4 + (g >> 1)) ^ rsw) << 1);
        auto frag = [&](int c) { return (c & 1 ? p1 : p0)[(c >> 1) * SY_R * 16]; };
        const double fa = frag(RA), fb = frag(RB);
#pragma unroll
        for (int c = RA; c < NR; c++) {
          const double bf = frag(c);
          sy_dmma(acc[c - RA][0], acc[c - RA][1], fa, bf);
          if (c >= RB) sy_dmma(acc[NR - RA + c - RB][0], acc[NR - RA + c - RB][1], fb, bf);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int f = 0; f < C::F; f++)
    *reinterpret_cast<double2*>(out + f * 64 + lane * 2) = make_double2(acc[f][0], acc[f][1]);
}

template <int NR, int... Ws>
__device__ __forceinline__ void sy_dispatch(int w, std::integer_sequence<int, Ws...>, const double* stg,
                                            unsigned long long* full, unsigned long long* empty, int64_t nchunks,
                                            int64_t cta, int64_t nct, double* out) {
  ((w == Ws ? sy_consume<NR, Ws>(stg, full, empty, nchunks, cta, nct, out) : void()), ...);
}

template <int NR>
__global__ void __launch_bounds__(SyCfg<NR>::THREADS, 1)
syrk_tma_kernel(const __grid_constant__ CUtensorMap tmA, int64_t rows, int nbox, double* __restrict__ part) {
  using C = SyCfg<NR>;
  extern __shared__ __align__(1024) unsigned char sy_raw[];
  unsigned char* base = sy_raw + ((1024u - (smem_u32(sy_raw) & 1023u)) & 1023u);
  double* stg = reinterpret_cast<double*>(base);  // [S][NB][SY_R][16], swizzled boxes
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + (size_t)C::S * C::STAGE);
  unsigned long long* empty = full + C::S;
  const int type = (int)(blockIdx.x % C::T);
  const int64_t cta = blockIdx.x / C::T, nct = gridDim.x / C::T;
  const int64_t nchunks = ceil_div<int64_t>(rows, SY_R);
  const int wp = warp_id(), lane = lane_id();
  if (threadIdx.x < C::S) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], C::CW);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (wp == C::CW) {  // ---------------- producer
    if (lane != 0) return;
    uint32_t q = 0;
    for (int64_t ch = cta; ch < nchunks; ch += nct, q++) {
      const int s = (int)(q % C::S);
      if (q >= C::S) mbar_wait(&empty[s], ((q / C::S) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[s])),
                   "r"((uint32_t)(nbox * SY_R * 128))
                   : "memory");
      for (int b = 0; b < nbox; b++)
        sy_tma(stg + ((size_t)s * C::NB + b) * SY_R * 16, &tmA, 16 * b, (int)(ch * SY_R), &full[s]);
    }
    return;
  }
  double* out = part + (size_t)blockIdx.x * C::PART + (size_t)wp * C::F * 64;
  sy_dispatch<NR>(type * C::CW + wp, std::make_integer_sequence<int, C::NW>{}, stg, full, empty, nchunks, cta, nct,
                  out);
}

// G[i][j] = G[j][i] (i <= j) = the partials of fragment (i/8, j/8) summed over its CTA type's
// CTAs in increasing order
template <int NR>
__global__ void syrk_reduce_kernel(const double* __restrict__ part, int nct, int n, double* __restrict__ G) {
  using C = SyCfg<NR>;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    if (i > j) continue;
    const int r = i >> 3, c = j >> 3;
    const int w = r < NR - 1 - r ? r : NR - 1 - r;
    const int type = w / C::CW, wl = w % C::CW;
    const int f = r == w ? c - w : NR - w + (c - (NR - 1 - w));
    const int idx = ((i & 7) * 4 + ((j & 7) >> 1)) * 2 + (j & 1);
    const double* p = part + (size_t)type * C::PART + (size_t)wl * C::F * 64 + (size_t)f * 64 + idx;
    double s = 0.0;
    for (int k = 0; k < nct; k++) s += p[(size_t)k * C::T * C::PART];
    G[(int64_t)i * n + j] = s;
    G[(int64_t)j * n + i] = s;
  }
}

template <int NR>
int sy_grid() {
  int dev = 0, sms = 148, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, syrk_tma_kernel<NR>, SyCfg<NR>::THREADS, SyCfg<NR>::SMEM) !=
          cudaSuccess ||
      per < 1)
    per = 1;
  const int T = SyCfg<NR>::T;
  return std::max(T, (std::min(sms * per, kSyMaxGrid) / T) * T);
}

template <int NR>
cudaError_t syrk_go(const double* A, int64_t lda, int64_t rows, int n, double* part, double* G, cudaStream_t st,
                    bool* done) {
  using C = SyCfg<NR>;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return cudaSuccess;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
  const cuuint32_t box[2] = {16, SY_R};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaSuccess;
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, syrk_tma_kernel<NR>, (int)C::SMEM)) return e;
  const int grid = sy_grid<NR>();
  note_launch();
  *done = true;
  cudaError_t e = launch_pdl(syrk_tma_kernel<NR>, dim3((unsigned)grid), dim3(C::THREADS), C::SMEM, st, map, rows,
                             (n + 15) / 16, part);
  if (e) return e;
  const int64_t total = (int64_t)n * n;
  note_launch();
  syrk_reduce_kernel<NR><<<(int)std::min<int64_t>(ceil_div<int64_t>(total, 256), 1024), 256, 0, st>>>(
      part, grid / C::T, n, G);
  return cudaGetLastError();
}

}  // namespace

size_t syrk_partials_bytes(int n) {
  if (n > 256) return 0;
  const size_t per = n <= 64 ? SyCfg<8>::PART : n <= 128 ? SyCfg<16>::PART : SyCfg<32>::PART;
  return (size_t)kSyMaxGrid * per * sizeof(double);
}

// G = A^T A through syrk_tma_kernel when A is TMA-describable and n <= 256 (*done), else the
// caller uses gram_kernel.  `part` holds syrk_partials_bytes(n).
cudaError_t launch_syrk(const double* A, int64_t lda, int64_t rows, int n, double* part, double* G, cudaStream_t st,
                        bool* done) {
  *done = false;
  static const bool on = [] { const char* e = getenv("RLHC_SYRK"); return !e || atoi(e) != 0; }();
  if (!on || n > 256 || n < 1 || rows < 1 || rows >= (int64_t(1) << 31) || (lda & 1) ||
      (reinterpret_cast<uintptr_t>(A) & 15))
    return cudaSuccess;
  if (n <= 64) return syrk_go<8>(A, lda, rows, n, part, G, st, done);
  if (n <= 128) return syrk_go<16>(A, lda, rows, n, part, G, st, done);
  return syrk_go<32>(A, lda, rows, n, part, G, st, done);
}

}  // namespace rlhc
