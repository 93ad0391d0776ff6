// tsgemm.cu -- the tall-skinny FP64 tensor-core product engine of the streaming stages:
//   C (rows x N) = Cin -/+ A (rows x K) B (K x N),   A streamed from HBM, B small (L2)
// used for the blocked left-looking Schur complements of the LU (C = X - L U, the fma chain
// of the elimination in increasing k: bitwise, DMMA m8n8k4 is the fma chain over its 4 k's,
// profiles/r01_probe_fp64_hbm.txt) and for the CholeskyQR products V = W D^-1, Q = V J^-1
// with B upper triangular (R#9: D, J have kappa <= ~7, so the explicit inverse is
// safe there; W = X Y^-1 stays a substitution).
//
// Persistent CTAs, one per SM; a CTA owns whole 128-row tiles and computes their 64-column
// blocks in DESCENDING order, so the row tile of A is read from HBM once (the other blocks
// hit L2) and, for triangular B, C may overwrite A in place (block j writes columns
// [64j, 64j+64), which the remaining blocks j' < j never read).
// Warp-specialised TMA pipeline: one elected thread of warp 8 (the PRODUCER) moves each
// 16-deep k chunk into one of S shared-memory stages -- the A tile (128 rows x 16 k) by a
// 2-D TMA copy (cp.async.bulk.tensor, 128-byte swizzle), the B tile (16 k x 64 columns)
// by a 1-D bulk copy of its pre-packed, padded image (pack_b_kernel) -- both completing on
// the stage's `full` mbarrier (expect_tx); warps 0-7 are CONSUMERS (32 x 32 DMMA tiles:
// wait `full`, compute, arrive on `empty`).  No CTA-wide barrier, no load code in the
// consumers, and the chunk sequence runs across tiles, so the next tile's chunks stream in
// during the current tile's epilogue.  A fragment row g of fragment a is tile row
// 16 (a/2) + 2 g + (a%2): with the 128-byte swizzle (16-byte chunk ^ row % 8) every
// fragment load is then bank-conflict free.  When A cannot be described to the TMA unit
// (odd lda, misaligned base) the producer warp writes the same swizzled layout with
// cp.async.  Measured history: every thread loading with one __syncthreads per chunk held
// the DMMA pipe at 70 % (the load phases coincided); a cp.async producer warp starved the
// consumers (20 % of their samples waiting on `full`); tools/probe/pdmma.cu shows the
// smem-fed 4 x 4 fragment loop itself at 99 % of the DMMA peak.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {
namespace {

constexpr int TG_M = 128;              // tile rows (4 x 2 consumer warps of 32 x 32)
constexpr int TG_N = 64;               // column block
constexpr int TG_K = 16;               // k chunk (128 bytes: one swizzled row)
constexpr int TG_S = 6;                // pipeline stages
constexpr int TG_BS = TG_N + 4;        // packed B row stride (doubles): conflict-free fragment loads
constexpr int TG_CW = 8;               // consumer warps
constexpr int TG_THREADS = 32 * (TG_CW + 1);
constexpr uint32_t TG_ABYTES = TG_M * TG_K * 8;     // 16 KB
constexpr uint32_t TG_BBYTES = TG_K * TG_BS * 8;    // 8704 B

struct __align__(1024) TgSmem {
  double A[TG_S][TG_M][TG_K];   // 128-byte rows, 16-byte chunks swizzled by row % 8
  double B[TG_S][TG_K][TG_BS];
  unsigned long long full[TG_S], empty[TG_S];
};
// element (row, k) of a swizzled A stage
__device__ __forceinline__ int a_off(int row, int k) { return row * TG_K + ((((k >> 1) ^ row) & 7) << 1) + (k & 1); }
// DMMA without `volatile`, so the compiler may schedule the fragment loads around it
__device__ __forceinline__ void dmma_s(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
// arrive on `bar` when this thread's cp.async copies issued so far have landed
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

struct TgArgs {
  const double* Bp;   // packed B: [ncb][nkc][TG_K][TG_BS] (pack_b_kernel)
  int nkc;            // k chunks per column block in the packed image
  const double* Cin;  // nullable: zero
  int64_t ldci;
  double* Cout;
  int64_t ldco;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  int64_t rows;
  int K, N;
  int ncb;            // column blocks
  int64_t nrt;        // row tiles
  unsigned long long* status;  // nullable: report non-finite Cin elements (input check)
  int n_index, col0;           // ... as ENONFINITE(INPUT, row * n_index + col0 + column)
};

// chunk sequence of this CTA: row tiles r = blockIdx.x + i * gridDim.x, each with its column
// blocks j = ncb-1 .. 0, each with chunks c = 0 .. nk-1 (blocks with nk = 0 only when K = 0)
template <bool TRI>
struct TgIter {
  int64_t r;
  int j, c, nk;
  __device__ void set_block(const TgArgs& p) {
    c = 0;
    const int kmax = TRI ? min(p.K, (j + 1) * TG_N) : p.K;
    nk = (kmax + TG_K - 1) / TG_K;
  }
  __device__ void start(const TgArgs& p, int64_t row_tile) {
    r = row_tile;
    j = p.ncb - 1;
    if (r < p.nrt) set_block(p);
  }
  __device__ bool valid(const TgArgs& p) const { return r < p.nrt; }
  __device__ void next_block(const TgArgs& p) {
    if (--j >= 0) set_block(p);
    else start(p, r + gridDim.x);
  }
};

// fallback producer (A not TMA-describable): the warp copies the A tile into the same
// swizzled layout with cp.async, lane 0 bulk-copies B; all arrive on `full` (33 arrivals)
__device__ __forceinline__ void tg_load_cp(const TgArgs& p, TgSmem& sm, int stage, int64_t r, int c) {
  const int64_t r0 = r * TG_M;
  const int kc = c * TG_K;
  const int lane = lane_id();
#pragma unroll 4
  for (int i = 0; i < TG_M * TG_K / 2 / 32; i++) {
    const int idx = lane + 32 * i;
    const int rr = idx >> 3, k2 = 2 * (idx & 7);
    const int64_t gr = r0 + rr;
    const int k = kc + k2;
    double* dst = &sm.A[stage][0][0] + a_off(rr, k2);
    const double* src = p.A + gr * p.lda + k;
    const bool rok = gr < p.rows;
    cp_async8(dst, (rok && k < p.K) ? src : p.A, (rok && k < p.K) ? 8 : 0);
    cp_async8(dst + 1, (rok && k + 1 < p.K) ? src + 1 : p.A, (rok && k + 1 < p.K) ? 8 : 0);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

template <bool TRI, bool SUB, bool TMA>
__global__ void __launch_bounds__(TG_THREADS, 1) ts_gemm_kernel(const __grid_constant__ CUtensorMap tmA, TgArgs p) {
  extern __shared__ __align__(1024) unsigned char tg_raw[];
  // 1024-byte alignment (128-byte swizzle) by an offset into the shared array, so that every
  // access below stays a shared-window access (LDS), not a generic one
  TgSmem& sm = *reinterpret_cast<TgSmem*>(tg_raw + ((1024u - (smem_u32(tg_raw) & 1023u)) & 1023u));
  const int lane = lane_id(), wp = warp_id();
  if (threadIdx.x < TG_S) {
    // TMA: one expect_tx arrival; cp.async fallback: 32 lane arrivals + lane 0's expect_tx
    mbar_init(&sm.full[threadIdx.x], TMA ? 1 : 33);
    mbar_init(&sm.empty[threadIdx.x], TG_CW);  // one arrival per consumer warp
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  TgIter<TRI> it;
  it.start(p, blockIdx.x);
  if (wp == TG_CW) {
    // ---------------- producer
    if (TMA && lane != 0) return;
    uint32_t q = 0;  // chunk counter
    while (it.valid(p)) {
      for (; it.c < it.nk; it.c++, q++) {
        const int s = (int)(q % TG_S);
        if (q >= TG_S) mbar_wait(&sm.empty[s], ((q / TG_S) - 1) & 1);
        const double* bsrc = p.Bp + ((size_t)it.j * p.nkc + it.c) * (TG_K * TG_BS);
        if (TMA) {
          mbar_expect_tx(&sm.full[s], TG_ABYTES + TG_BBYTES);
          tma_2d(&sm.A[s][0][0], &tmA, it.c * TG_K, (int)(it.r * TG_M), &sm.full[s]);
          bulk_g2s(&sm.B[s][0][0], bsrc, TG_BBYTES, &sm.full[s]);
        } else {
          if (lane == 0) {
            mbar_expect_tx(&sm.full[s], TG_BBYTES);
            bulk_g2s(&sm.B[s][0][0], bsrc, TG_BBYTES, &sm.full[s]);
          }
          tg_load_cp(p, sm, s, it.r, it.c);
          cp_async_mbar_arrive(&sm.full[s]);
        }
      }
      it.next_block(p);
    }
    if (!TMA) asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }
  // ---------------- consumers: warp = 32 rows x 32 columns (4 x 4 fragments); fragment a's
  // row g is tile row wi + 16 (a/2) + 2 g + (a%2) (conflict-free against the swizzle)
  const int g = lane >> 2, tq = lane & 3;
  const int wi = (wp >> 1) * 32, wj = (wp & 1) * 32;
  auto frow = [&](int a) { return wi + 16 * (a >> 1) + 2 * g + (a & 1); };
  const bool st16 = ((p.ldco & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.Cout) & 15) == 0);
  uint32_t q = 0;
  double acc[4][4][2];
  while (it.valid(p)) {
    const int64_t r0 = it.r * TG_M;
    const int c0 = it.j * TG_N;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int64_t gr = r0 + frow(a);
        const int c = c0 + wj + b * 8 + 2 * tq;
        if (p.Cin && gr < p.rows) {  // plain loads: Cin may be Cout (in place)
          acc[a][b][0] = c < p.N ? p.Cin[gr * p.ldci + c] : 0.0;
          acc[a][b][1] = c + 1 < p.N ? p.Cin[gr * p.ldci + c + 1] : 0.0;
          if (p.status) {
            if (!isfinite(acc[a][b][0]))
              report(p.status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, gr * p.n_index + p.col0 + c);
            if (!isfinite(acc[a][b][1]))
              report(p.status, RLHC_ENONFINITE, RLHC_STAGE_INPUT, gr * p.n_index + p.col0 + c + 1);
          }
        } else {
          acc[a][b][0] = acc[a][b][1] = 0.0;
        }
      }
    for (; it.c < it.nk; it.c++, q++) {
      const int s = (int)(q % TG_S);
      mbar_wait(&sm.full[s], (q / TG_S) & 1);
      // triangular B: this warp's columns [c0 + wj, c0 + wj + 32) need k < c0 + wj + 32 only,
      // and in the two chunks on the warp's diagonal (d = k - (c0 + wj) = 0 or 16) fragment b
      // (columns c0 + wj + 8 b ..) only k <= c0 + wj + 8 b + 7: B is exactly zero below that, so
      // those steps would only add signed zeros
      const int dk = it.c * TG_K - (c0 + wj);
      if (TRI && (dk == 0 || dk == 16)) {
#pragma unroll
        for (int k0 = 0; k0 < TG_K; k0 += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int a = 0; a < 4; a++) {
            const double v = (&sm.A[s][0][0])[a_off(frow(a), k0 + tq)];
            af[a] = SUB ? -v : v;
          }
#pragma unroll
          for (int b = 0; b < 4; b++) bf[b] = sm.B[s][k0 + tq][wj + b * 8 + g];
          if (dk == 0) {
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
              for (int b = 0; b < 4; b++)
                if (k0 <= 8 * b + 7) dmma_s(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
          } else {
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
              for (int b = 0; b < 4; b++)
                if (16 + k0 <= 8 * b + 7) dmma_s(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
          }
        }
      } else if (!TRI || dk < 32) {
#pragma unroll
        for (int k0 = 0; k0 < TG_K; k0 += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int a = 0; a < 4; a++) {
            const double v = (&sm.A[s][0][0])[a_off(frow(a), k0 + tq)];
            af[a] = SUB ? -v : v;
          }
#pragma unroll
          for (int b = 0; b < 4; b++) bf[b] = sm.B[s][k0 + tq][wj + b * 8 + g];
#pragma unroll
          for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) dmma_s(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int64_t gr = r0 + frow(a);
        const int c = c0 + wj + b * 8 + 2 * tq;
        if (gr < p.rows) {
          double* dst = p.Cout + gr * p.ldco + c;
          if (st16 && c + 1 < p.N) {
            *reinterpret_cast<double2*>(dst) = make_double2(acc[a][b][0], acc[a][b][1]);
          } else {
            if (c < p.N) dst[0] = acc[a][b][0];
            if (c + 1 < p.N) dst[1] = acc[a][b][1];
          }
        }
      }
    it.next_block(p);
  }
}


// B (K x N, ldb) -> [ncb][nkc][16][68] (zero-padded), the image each stage bulk-copies
__global__ void pack_b_kernel(const double* __restrict__ B, int64_t ldb, int K, int N, int ncb, int nkc,
                              double* __restrict__ Bp) {
  const int64_t total = (int64_t)ncb * nkc * TG_K * TG_BS;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int cc = (int)(e % TG_BS);
    const int64_t rest = e / TG_BS;
    const int kk = (int)(rest % TG_K);
    const int64_t jc = rest / TG_K;
    const int c = (int)(jc % nkc), j = (int)(jc / nkc);
    const int k = c * TG_K + kk, col = j * TG_N + cc;
    Bp[e] = (cc < TG_N && k < K && col < N) ? B[(int64_t)k * ldb + col] : 0.0;
  }
}

template <bool TRI, bool SUB, bool TMA>
cudaError_t ts_gemm_launch(const CUtensorMap& map, const TgArgs& p, cudaStream_t st) {
  constexpr int smem = (int)sizeof(TgSmem) + 1024;  // + alignment slack (128-byte swizzle: 1 KB)
  static DevFlags attr;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if ((e = smem_attr(attr, ts_gemm_kernel<TRI, SUB, TMA>, smem))) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p.nrt, (int64_t)sms));
  note_launch();
  return launch_pdl(ts_gemm_kernel<TRI, SUB, TMA>, dim3((unsigned)grid), dim3(TG_THREADS), (size_t)smem, st, map, p);
}

template <bool TRI, bool SUB>
cudaError_t ts_gemm_go(const TgArgs& p, cudaStream_t st) {
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  const bool tma = enc && (p.lda % 2) == 0 && (reinterpret_cast<uintptr_t>(p.A) & 15) == 0 && p.K >= 1;
  if (tma) {
    const cuuint64_t dims[2] = {(cuuint64_t)p.K, (cuuint64_t)p.rows};
    const cuuint64_t strides[1] = {(cuuint64_t)p.lda * 8};
    const cuuint32_t box[2] = {TG_K, TG_M};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.A), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) return ts_gemm_launch<TRI, SUB, true>(map, p, st);
  }
  return ts_gemm_launch<TRI, SUB, false>(map, p, st);
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// Cout = Cin - A B (sub) or Cin + A B; Cin nullable (zero); B upper triangular when tri
// (B[k][c] = 0 for k > c is never read).  Cout may alias Cin (each tile reads its Cin before
// writing it, tiles are disjoint).  Cout may alias A only when tri and K == N (in-place
// triangular product: the descending column blocks never read what they overwrote).
size_t ts_gemm_pack_bytes(int K, int N) {
  return std::max((size_t)ceil_div(N, TG_N) * ceil_div(std::max(K, 1), TG_K) * TG_K * TG_BS * sizeof(double),
                  K == N ? tri_pack_bytes(N) : (size_t)0);
}

cudaError_t launch_ts_gemm_checked_impl(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                                        int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N,
                                        bool tri, bool sub, double* bpack, unsigned long long* status, int n_index,
                                        int col0, cudaStream_t st);

cudaError_t launch_ts_gemm(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A, int64_t lda,
                           const double* B, int64_t ldb, int64_t rows, int K, int N, bool tri, bool sub, double* bpack,
                           cudaStream_t st) {
  return launch_ts_gemm_checked_impl(Cin, ldci, Cout, ldco, A, lda, B, ldb, rows, K, N, tri, sub, bpack, nullptr, 0,
                                     0, st);
}

cudaError_t launch_ts_gemm_checked(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                                   int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N, double* bpack,
                                   unsigned long long* status, int n_index, int col0_index, cudaStream_t st) {
  return launch_ts_gemm_checked_impl(Cin, ldci, Cout, ldco, A, lda, B, ldb, rows, K, N, false, true, bpack, status,
                                     n_index, col0_index, st);
}

cudaError_t launch_ts_gemm_checked_impl(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                                        int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N,
                                        bool tri, bool sub, double* bpack, unsigned long long* status, int n_index,
                                        int col0, cudaStream_t st) {
  if (rows <= 0 || N <= 0) return cudaSuccess;
  if (tri && !sub && !Cin && K == N) {  // the in-place CholeskyQR products: trmm.cu
    bool done = false;
    if (cudaError_t e = launch_tri_tma(A, lda, B, ldb, rows, N, Cout, ldco, bpack, st, &done)) return e;
    if (done) return cudaSuccess;
  }
  TgArgs p{bpack, ceil_div(std::max(K, 1), TG_K), Cin, ldci, Cout, ldco, A, lda, B, ldb, rows, K, N, 0, 0,
           status, n_index, col0};
  p.ncb = ceil_div(N, TG_N);
  p.nrt = ceil_div<int64_t>(rows, TG_M);
  const int64_t total = (int64_t)p.ncb * p.nkc * TG_K * TG_BS;
  note_launch();
  pack_b_kernel<<<(unsigned)std::min<int64_t>(ceil_div<int64_t>(total, 256), 1024), 256, 0, st>>>(B, ldb, K, N, p.ncb,
                                                                                                    p.nkc, bpack);
  if (cudaError_t e = cudaGetLastError()) return e;
  if (tri) return sub ? ts_gemm_go<true, true>(p, st) : ts_gemm_go<true, false>(p, st);
  return sub ? ts_gemm_go<false, true>(p, st) : ts_gemm_go<false, false>(p, st);
}

}  // namespace rlhc
