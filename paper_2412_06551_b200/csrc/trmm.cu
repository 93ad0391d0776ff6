// trmm.cu -- C = A B with B upper triangular (n x n, 64 < n <= 256), A streamed (rows >> n),
// C may overwrite A: the CholeskyQR products V = W D^-1 and Q = V J^-1 (D^-1, J^-1
// formed explicitly, R#9) as a column-balanced, TMA-fed DMMA pipeline.
//
// Output columns come in NR = n / 8 fragment columns (rounded up to 16, 32 or 64); column
// fragment c needs the k4 steps s <= 2 c + 1 only (B is zero below its diagonal), so the
// columns c and NR/2-1-c ... are paired as in syrk.cu: warp w owns the column fragments
// {16 p + w, 16 p + 15 - w} (p < NR / 16) -- every warp the same number of DMMAs -- and every
// row of the tile (NRF row fragments, 32 fragments per warp).  One CTA per SM (8 consumer
// warps at 232 registers by setmaxnreg, one producer thread), persistent over R-row tiles (R = 8 NRF).  Per 16-deep k chunk
// the producer moves A's R x 16 tile by a 2-D TMA copy (128-byte swizzle) and B's chunk --
// pre-packed in DMMA fragment order (pack_tri_kernel: only the column fragments the chunk
// feeds, lane-contiguous, so each fragment load is one conflict-free 256-byte read) -- by one
// 1-D bulk copy, both on the stage's `full` mbarrier; consumers release `empty`.  A row of
// fragment a is tile row 16 (a / 2) + 2 g + (a % 2) (conflict-free against the swizzle, as in
// tsgemm.cu).  Per output element the k terms are accumulated in increasing k with the same
// DMMAs as ts_gemm_kernel's triangular product (the same k4 steps skipped), so the result is
// bit-identical to it.  Stores go straight from the accumulators after the tile's last chunk;
// in place is safe because every chunk of a tile has landed in shared memory before any
// warp stores that tile's rows, and tiles are disjoint.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {
namespace {

template <int NR>
struct TrCfg {
  static constexpr int NCW = NR / 8;           // column fragments per warp
  static constexpr int NRF = 32 / NCW;         // row fragments per warp (= per tile)
  static constexpr int R = 8 * NRF;            // tile rows
  static constexpr int NKC = NR / 2;           // 16-deep k chunks
  static constexpr uint32_t ABYTES = R * 128;  // A box: R rows x 16 k
  static constexpr uint32_t BMAX = 4 * NR * 256;
  static constexpr uint32_t STAGE = ABYTES + BMAX;
  static constexpr int S = (220 * 1024) / STAGE > 6 ? 6 : (220 * 1024) / STAGE;
  static constexpr int THREADS = 32 * 12;  // 2 consumer warpgroups + the producer's
  static constexpr size_t SMEM = (size_t)S * STAGE + 2 * S * 8 + 1024;
};
// packed B: chunk kc holds [4 k4 steps][NR - 2 kc column fragments][32 lanes]
__host__ __device__ inline size_t tri_chunk_off(int NR, int kc) {  // doubles before chunk kc
  return (size_t)128 * ((size_t)NR * kc - (size_t)kc * (kc - 1));
}
__host__ __device__ inline int tri_nr(int n) { return n <= 128 ? 16 : n <= 256 ? 32 : 64; }

__global__ void pack_tri_kernel(const double* __restrict__ B, int64_t ldb, int n, int NR, double* __restrict__ Bp) {
  const size_t total = tri_chunk_off(NR, NR / 2);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int kc = 0;
    while (tri_chunk_off(NR, kc + 1) <= e) kc++;
    const size_t r = e - tri_chunk_off(NR, kc);
    const int nc = NR - 2 * kc;
    const int lane = (int)(r & 31), cc = (int)((r >> 5) % nc), s = (int)((r >> 5) / nc);
    const int k = 16 * kc + 4 * s + (lane & 3), col = 8 * (2 * kc + cc) + (lane >> 2);
    Bp[e] = (k < n && col < n && k <= col) ? B[(int64_t)k * ldb + col] : 0.0;
  }
}

__device__ __forceinline__ void tr_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ int tr_aoff(int row, int k) { return row * 16 + ((((k >> 1) ^ row) & 7) << 1) + (k & 1); }

// The k4 steps a column fragment skips are decided per 16-deep chunk: column fragment c takes
// part in chunk kc iff c >= 2 kc (so its diagonal chunk adds two k4 steps of exact zeros), and
// a warp's fragments are in increasing order, so the active ones are a suffix [i0, NCW): one
// straight-line body per i0 (chunk_body<I0>), selected once per chunk.  (A branch per k4 step
// and column fragment split the DMMA stream into blocks the scheduler could not interleave.)
template <int NR, int I0>
__device__ __forceinline__ void tr_chunk(const double* As, const double* Bs, int nc, int kc, int W, int lane,
                                         int g, int t, double (&acc)[TrCfg<NR>::NRF][TrCfg<NR>::NCW][2]) {
  using G = TrCfg<NR>;
  auto colf = [&](int i) { return 16 * (i >> 1) + ((i & 1) ? 15 - W : W); };
  auto frow = [&](int a) { return 16 * (a >> 1) + 2 * g + (a & 1); };
  int boff[G::NCW];
#pragma unroll
  for (int i = I0; i < G::NCW; i++) boff[i] = (colf(i) - 2 * kc) * 32 + lane;
#pragma unroll
  for (int s4 = 0; s4 < 4; s4++) {
    double af[G::NRF], bf[G::NCW];
#pragma unroll
    for (int a = 0; a < G::NRF; a++) af[a] = As[tr_aoff(frow(a), 4 * s4 + t)];
#pragma unroll
    for (int i = I0; i < G::NCW; i++) bf[i] = Bs[s4 * nc * 32 + boff[i]];
#pragma unroll
    for (int i = I0; i < G::NCW; i++)
#pragma unroll
      for (int a = 0; a < G::NRF; a++) tr_dmma(acc[a][i][0], acc[a][i][1], af[a], bf[i]);
  }
}
template <int NR, int... Is>
__device__ __forceinline__ void tr_chunk_sel(int i0, std::integer_sequence<int, Is...>, const double* As,
                                             const double* Bs, int nc, int kc, int W, int lane, int g, int t,
                                             double (&acc)[TrCfg<NR>::NRF][TrCfg<NR>::NCW][2]) {
  ((i0 == Is ? tr_chunk<NR, Is>(As, Bs, nc, kc, W, lane, g, t, acc) : void()), ...);
}

template <int NR>
__device__ __forceinline__ void tr_consume(int W, const unsigned char* stg, unsigned long long* full,
                                           unsigned long long* empty, int64_t rows, int n, int64_t ntiles,
                                           double* __restrict__ C, int64_t ldc) {
  using G = TrCfg<NR>;
  const int lane = lane_id(), g = lane >> 2, t = lane & 3;
  auto colf = [&](int i) { return 16 * (i >> 1) + ((i & 1) ? 15 - W : W); };
  auto frow = [&](int a) { return 16 * (a >> 1) + 2 * g + (a & 1); };
  const bool st16 = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  uint32_t q = 0;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    double acc[G::NRF][G::NCW][2];
#pragma unroll
    for (int a = 0; a < G::NRF; a++)
#pragma unroll
      for (int i = 0; i < G::NCW; i++) acc[a][i][0] = acc[a][i][1] = 0.0;
#pragma unroll 1
    for (int kc = 0; kc < G::NKC; kc++, q++) {
      const int s = (int)(q % G::S);
      mbar_wait(&full[s], (q / G::S) & 1);
      const double* As = reinterpret_cast<const double*>(stg + (size_t)s * G::STAGE);
      const double* Bs = reinterpret_cast<const double*>(stg + (size_t)s * G::STAGE + G::ABYTES);
      int i0 = 0;
#pragma unroll
      for (int i = 0; i < G::NCW; i++) i0 += colf(i) < 2 * kc;
      tr_chunk_sel<NR>(i0, std::make_integer_sequence<int, G::NCW>{}, As, Bs, NR - 2 * kc, kc, W, lane, g, t, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    const int64_t r0 = tl * G::R;
#pragma unroll
    for (int a = 0; a < G::NRF; a++) {
      const int64_t gr = r0 + frow(a);
      if (gr >= rows) continue;
#pragma unroll
      for (int i = 0; i < G::NCW; i++) {
        const int col = 8 * colf(i) + 2 * t;
        double* dst = C + gr * ldc + col;
        if (st16 && col + 1 < n) {
          *reinterpret_cast<double2*>(dst) = make_double2(acc[a][i][0], acc[a][i][1]);
        } else {
          if (col < n) dst[0] = acc[a][i][0];
          if (col + 1 < n) dst[1] = acc[a][i][1];
        }
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(TrCfg<NR>::THREADS, 1)
tri_tma_kernel(const __grid_constant__ CUtensorMap tmA, const double* __restrict__ Bp, int64_t rows, int n,
               double* __restrict__ C, int64_t ldc) {
  using G = TrCfg<NR>;
  extern __shared__ __align__(1024) unsigned char tr_raw[];
  unsigned char* stg = tr_raw + ((1024u - (smem_u32(tr_raw) & 1023u)) & 1023u);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(stg + (size_t)G::S * G::STAGE);
  unsigned long long* empty = full + G::S;
  const int64_t ntiles = ceil_div<int64_t>(rows, G::R);
  const int wp = warp_id(), lane = lane_id();
  if (threadIdx.x < G::S) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], 8);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (wp >= 8) {  // ---------------- producer warpgroup: one thread works
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (wp != 8 || lane != 0) return;
    uint32_t q = 0;
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x)
      for (int kc = 0; kc < G::NKC; kc++, q++) {
        const int s = (int)(q % G::S);
        if (q >= G::S) mbar_wait(&empty[s], ((q / G::S) - 1) & 1);
        const uint32_t bbytes = 4u * (uint32_t)(NR - 2 * kc) * 256u;
        unsigned long long* bar = &full[s];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                     "r"(G::ABYTES + bbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];\n" ::"r"(smem_u32(stg + (size_t)s * G::STAGE)),
            "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(16 * kc), "r"((int)(tl * G::R)), "r"(smem_u32(bar))
            : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(stg + (size_t)s * G::STAGE + G::ABYTES)),
                     "l"(Bp + tri_chunk_off(NR, kc)), "r"(bbytes), "r"(smem_u32(bar))
                     : "memory");
      }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");  // 8 x 32 x 232 + 4 x 32 x 40 <= 64K
  tr_consume<NR>(wp, stg, full, empty, rows, n, ntiles, C, ldc);
}

template <int NR>
cudaError_t tri_go(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int n, double* C,
                   int64_t ldc, double* bpack, cudaStream_t st, bool* done) {
  using G = TrCfg<NR>;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return cudaSuccess;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)G::R};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaSuccess;
  static DevFlags attr;
  if (cudaError_t e = smem_attr(attr, tri_tma_kernel<NR>, (int)G::SMEM)) return e;
  const size_t total = tri_chunk_off(NR, NR / 2);
  note_launch();
  pack_tri_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 1024), 256, 0, st>>>(B, ldb, n, NR, bpack);
  if (cudaError_t e = cudaGetLastError()) return e;
  int dev = 0, sms = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  if (cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(rows, G::R), sms));
  note_launch();
  *done = true;
  return launch_pdl(tri_tma_kernel<NR>, dim3((unsigned)grid), dim3(G::THREADS), G::SMEM, st, map,
                    (const double*)bpack, rows, n, C, ldc);
}

}  // namespace

size_t tri_pack_bytes(int n) {
  if (n <= 64 || n > 256) return 0;
  const int NR = tri_nr(n);
  return tri_chunk_off(NR, NR / 2) * sizeof(double);
}

// C = A B, B upper triangular n x n (64 < n <= 512), through tri_tma_kernel when A is
// TMA-describable (*done); C may be A.  bpack: tri_pack_bytes(n) bytes of scratch.
cudaError_t launch_tri_tma(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int n, double* C,
                           int64_t ldc, double* bpack, cudaStream_t st, bool* done) {
  *done = false;
  static const bool on = [] { const char* e = getenv("RLHC_TRI_TMA"); return !e || atoi(e) != 0; }();
  // n <= 256 with at least 8 tiles per SM: measured faster than ts_gemm_kernel there (cfg5 V
  // pass 40.9 -> 37.6 ms, cfg3 0.99 -> 0.85 ms); at n = 512 the two tie (3.0 ms at 262144 rows)
  // and for short A the 64-row tiles leave a ragged last wave
  if (!on || n <= 64 || n > 256 || rows < 1 || rows >= (int64_t(1) << 31) || (lda & 1) ||
      (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(bpack) & 15))
    return cudaSuccess;
  const int NR = tri_nr(n);
  if (ceil_div<int64_t>(rows, NR == 16 ? TrCfg<16>::R : TrCfg<32>::R) < 8 * 148) return cudaSuccess;
  if (NR == 16) return tri_go<16>(A, lda, B, ldb, rows, n, C, ldc, bpack, st, done);
  return tri_go<32>(A, lda, B, ldb, rows, n, C, ldc, bpack, st, done);
}

}  // namespace rlhc
