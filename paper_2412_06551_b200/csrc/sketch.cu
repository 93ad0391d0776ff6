// sketch.cu -- the sketches of the L factor ("L_s = Omega L",
// P:294 "L_ss = Omega_2 Omega_1 L"):
//   * Gaussian: out = Omega A with Omega generated in-kernel from Philox (never
//     stored), contracted on the FP64 tensor cores (DMMA), split over rows with a
//     fixed-order reduction of the partial tiles;
//   * CountSketch: deterministic bucket gather -- rows are stably sorted by bucket
//     (counting sort on the Philox hash) and each bucket is summed in ascending row
//     order, so the result is bitwise reproducible without floating atomics.
#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {

// ------------------------------------------------------------------ Gaussian
// CTA output tile: ST = 64 sketch rows x NT = 32*NTW columns, warps 2 x NTW (32 x 32 each,
// DMMA m8n8k4 fragments).  Per chunk of SK rows of A: the CTA generates the Omega tile
// (64 x SK, Philox + Box-Muller, R#19) while the next chunk's A tile streams in with
// cp.async (double buffer), then the DMMA contraction.  Omega is regenerated once per
// column tile, so n > 64 uses 256-column tiles (NTW = 8).  (Measured alternatives: 2 CTAs
// of 64 x 128 per SM, and warp-specialised generator warps feeding compute warps through
// mbarriers, were both slower: the Box-Muller generation is a latency-bound ~250-
// instruction chain per pair and needs every warp of the SM to keep up.)
constexpr int ST = 64;   // output tile rows (sketch rows)
constexpr int SK = 32;   // rows of A per chunk

static int gauss_ntw(int n) { return n <= 64 ? 2 : 8; }

struct GaussGeom {
  int ti, tj, nsplit, nt;
  int64_t rows_per_split;
};
static GaussGeom gauss_geom(int64_t rows, int n, int s) {
  GaussGeom g;
  g.nt = 32 * gauss_ntw(n);
  g.ti = ceil_div(s, ST);
  g.tj = ceil_div(n, g.nt);
  const int tiles = g.ti * g.tj;
  // resident CTAs: 2 per SM (64-column tiles, 128 threads) or 1 (256-column tiles, 512
  // threads); at least 2 waves, split count rounded so the last wave is (nearly) full
  const int64_t slots = (g.nt == 64 ? 2 : 1) * (int64_t)kSMs;
  int64_t want = std::max<int64_t>(1, (2 * slots + tiles - 1) / tiles);
  const int64_t waves = (want * tiles + slots - 1) / slots;
  want = std::max<int64_t>(1, waves * slots / tiles);
  int64_t maxs = std::max<int64_t>(1, rows / 128);
  g.nsplit = (int)std::min<int64_t>(want, maxs);
  g.rows_per_split = ceil_div<int64_t>(ceil_div<int64_t>(rows, g.nsplit), SK) * SK;
  g.nsplit = (int)std::max<int64_t>(1, ceil_div<int64_t>(rows, g.rows_per_split));
  return g;
}
size_t gauss_partials_bytes(int64_t rows, int n, int s) {
  GaussGeom g = gauss_geom(rows, n, s);
  return (size_t)g.nsplit * g.ti * g.tj * ST * g.nt * sizeof(double);
}

template <int NTW, bool OMEM>
struct GaussSmem {
  static constexpr int NT = 32 * NTW;
  double A[2][SK][NT + 4];            // A tile, double-buffered (row pad 4: conflict-free B fragments)
  double Om[OMEM ? 2 : 1][ST][SK + 4];  // Omega tile (row pad 4: conflict-free A fragments)
};

// Omega (s x cols, entries of stream `stream_id` scaled by 1/sqrt(s), exactly the values
// gauss_sketch_kernel generates) written to Om (row-major, ld ldom, rows rounded up to
// even; the pad row is zero).  Launched on a side stream so that the Box-Muller work
// overlaps the latency-bound TSLU; the sketch then streams Omega from HBM (OMEM).
__global__ void __launch_bounds__(256)
omega_gen_kernel(uint64_t seed, uint32_t stream_id, int s, int64_t cols, int64_t row0, double* __restrict__ Om,
                 int64_t ldom) {
  const double scale = __ddiv_rn(1.0, __dsqrt_rn((double)s));
  const int64_t total = (int64_t)((s + 1) / 2) * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ip = idx / cols, r = idx - ip * cols;
    double z0, z1;
    gauss_pair(seed, (uint64_t)(row0 + r), (uint32_t)ip, stream_id, &z0, &z1);
    Om[(2 * ip) * ldom + r] = __dmul_rn(z0, scale);
    Om[(2 * ip + 1) * ldom + r] = (2 * ip + 1 < s) ? __dmul_rn(z1, scale) : 0.0;
  }
}

template <int NTW, bool OMEM>
__global__ void __launch_bounds__(64 * NTW)
gauss_sketch_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int n, int64_t row0, int s,
                    uint64_t seed, uint32_t stream_id, int64_t rows_per_split, double* __restrict__ part,
                    const double* __restrict__ Omg, int64_t ldom) {
  constexpr int NT = 32 * NTW, NTH = 64 * NTW;
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GaussSmem<NTW, OMEM>& sm = *reinterpret_cast<GaussSmem<NTW, OMEM>*>(gsm_raw);
  const int tjn = (n + NT - 1) / NT;
  const int tile_i = blockIdx.x / tjn, tile_j = blockIdx.x % tjn;
  const int i0 = tile_i * ST, j0 = tile_j * NT;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = std::min<int64_t>(rows, r0 + rows_per_split);
  const double scale = __ddiv_rn(1.0, __dsqrt_rn((double)s));
  const int lane = lane_id(), w = warp_id();
  const int g = lane >> 2, t = lane & 3;
  const int wi = (w / NTW) * 32, wj = (w % NTW) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
  const bool aligned = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  // A tile (SK rows x NT columns) of the chunk at k0 into buffer b: 16-byte async copies
  // interior chunks: thread copies row (tid / (NT/2)) + j*(NTH/(NT/2)), one fixed column
  // pair -- no per-copy index arithmetic or bounds tests
  constexpr int RSTEP = NTH / (NT / 2);  // rows covered per pass (NT/2 threads per row)
  const bool cols_full = aligned && j0 + NT <= n;
  const int s_even = (s + 1) & ~1;  // rows of the stored Omega
  auto fetch = [&](int64_t k0, int b) {
    if (OMEM) {  // Omega tile rows i0..i0+63, columns k0..k0+SK-1 (zero outside s_even x r1)
      if (k0 + SK <= r1 && i0 + ST <= s_even) {
        const int rr = threadIdx.x / (SK / 2), cc = 2 * (threadIdx.x % (SK / 2));
        constexpr int OSTEP = NTH / (SK / 2);
#pragma unroll
        for (int j = 0; j < ST / OSTEP; j++)
          cp_async16(&sm.Om[b][rr + j * OSTEP][cc], Omg + (int64_t)(i0 + rr + j * OSTEP) * ldom + k0 + cc);
      } else {
        for (int idx = threadIdx.x; idx < ST * SK; idx += NTH) {
          const int ii = idx / SK, kk = idx - ii * SK;
          const bool in = i0 + ii < s_even && k0 + kk < r1;
          sm.Om[b][ii][kk] = in ? Omg[(int64_t)(i0 + ii) * ldom + k0 + kk] : 0.0;
        }
      }
    }
    if (cols_full && k0 + SK <= r1) {
      const int rr = threadIdx.x / (NT / 2), cc = 2 * (threadIdx.x % (NT / 2));
      const double* src = A + (k0 + rr) * lda + j0 + cc;
#pragma unroll
      for (int j = 0; j < SK / RSTEP; j++) cp_async16(&sm.A[b][rr + j * RSTEP][cc], src + (int64_t)j * RSTEP * lda);
      cp_async_commit();
      return;
    }
    for (int idx = threadIdx.x; idx < SK * (NT / 2); idx += NTH) {
      const int kk = idx / (NT / 2), c = 2 * (idx % (NT / 2));
      const int64_t gr = k0 + kk;
      double* dst = &sm.A[b][kk][c];
      const double* src = A + gr * lda + j0 + c;
      if (gr < r1 && aligned && j0 + c + 1 < n) cp_async16(dst, src);
      else {
        dst[0] = (gr < r1 && j0 + c < n) ? src[0] : 0.0;
        dst[1] = (gr < r1 && j0 + c + 1 < n) ? src[1] : 0.0;
      }
    }
    cp_async_commit();
  };
  if (r0 < r1) fetch(r0, 0);
  int buf = 0;
  for (int64_t k0 = r0; k0 < r1; k0 += SK, buf ^= 1) {
    // Omega tile: rows i0..i0+63 (pairs i, i+1 share one Philox block), columns k0..k0+SK-1
    for (int idx = threadIdx.x; !OMEM && idx < (ST / 2) * SK; idx += NTH) {
      int ip = idx / SK, kk = idx - ip * SK;
      int i = i0 + 2 * ip;
      int64_t gr = k0 + kk;
      double z0 = 0.0, z1 = 0.0;
      if (gr < r1 && i < s) {
        gauss_pair(seed, (uint64_t)(row0 + gr), (uint32_t)(i >> 1), stream_id, &z0, &z1);
        z0 = __dmul_rn(z0, scale);
        z1 = (i + 1 < s) ? __dmul_rn(z1, scale) : 0.0;
      }
      sm.Om[0][2 * ip][kk] = z0;
      sm.Om[0][2 * ip + 1][kk] = z1;
    }
    // next chunk's A tile into the other buffer (freed by the barrier that ended the
    // previous iteration), then wait for this chunk's tile only
    if (k0 + SK < r1) {
      fetch(k0 + SK, buf ^ 1);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = sm.Om[OMEM ? buf : 0][wi + a * 8 + g][kk + t];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = sm.A[buf][kk + t][wj + b * 8 + g];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
  double* P = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * ST * NT;
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) {
      int r = wi + a * 8 + g, c = wj + b * 8 + 2 * t;
      P[r * NT + c] = acc[a][b][0];
      P[r * NT + c + 1] = acc[a][b][1];
    }
}

// out = sum over the row splits of the partial tiles, in a fixed order: block = 32
// consecutive partial elements x 8 warps, warp q sums splits [q*per, (q+1)*per) with 8
// independent accumulators (loads in flight), then the 8 warp sums are combined in order.
__global__ void __launch_bounds__(256)
gauss_reduce_kernel(const double* __restrict__ part, int nsplit, int ntiles, int tjn, int nt, int n, int s,
                    double* __restrict__ out) {
  __shared__ double red[8][32];
  const int lane = lane_id(), wq = warp_id();
  const int64_t tile_sz = (int64_t)ST * nt;
  const int64_t per_split = (int64_t)ntiles * tile_sz;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int per = (nsplit + 7) / 8;
  const int p0 = wq * per, p1 = min(nsplit, p0 + per);
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (e < per_split) {
    const double* p = part + e;
    int q = p0;
    for (; q + 8 <= p1; q += 8)
#pragma unroll
      for (int u = 0; u < 8; u++) acc[u] += p[(size_t)(q + u) * per_split];
    for (; q < p1; q++) acc[0] += p[(size_t)q * per_split];
  }
  red[wq][lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (wq == 0 && e < per_split) {
    double v = red[0][lane];
    for (int q = 1; q < 8; q++) v += red[q][lane];
    const int tile = (int)(e / tile_sz), rc = (int)(e - (int64_t)tile * tile_sz);
    const int i = (tile / tjn) * ST + rc / nt, j = (tile % tjn) * nt + rc % nt;
    if (i < s && j < n) out[(int64_t)i * n + j] = v;
  }
}

int64_t omega_ld(int64_t cols) { return (cols + 3) & ~(int64_t)3; }
size_t omega_bytes(int64_t s, int64_t cols) { return (size_t)((s + 1) & ~(int64_t)1) * omega_ld(cols) * sizeof(double); }

cudaError_t launch_omega_gen(uint64_t seed, uint32_t stream_id, int s, int64_t cols, int64_t row0, double* Om,
                             cudaStream_t st) {
  const int64_t total = (int64_t)((s + 1) / 2) * cols;
  if (total == 0) return cudaSuccess;
  // full occupancy: fewer generator CTAs per SM only stretch its overlap with the TSLU
  // (measured cfg4a TSLU +2.2 ms at 1 CTA/SM, +1.4 ms at 8)
  static const int per_sm = [] {
    const char* e = getenv("RLHC_OMEGA_CTAS");
    return e ? atoi(e) : 8;
  }();
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), (int64_t)per_sm * kSMs);
  note_launch(); omega_gen_kernel<<<grid, 256, 0, st>>>(seed, stream_id, s, cols, row0, Om, omega_ld(cols));
  return cudaGetLastError();
}

cudaError_t launch_omega_gen_cols(uint64_t seed, int s, int64_t m, int64_t c0, int64_t ncols, double* Om,
                                  cudaStream_t st) {
  const int64_t total = (int64_t)((s + 1) / 2) * ncols;
  if (total <= 0) return cudaSuccess;
  // few CTAs per SM: the chunk shares the SMs with a latency-bound tournament, whose select
  // warps need the issue slots (RLHC_OMEGA_CHUNK_CTAS, measurement knob)
  static const int per_sm = [] {
    const char* e = getenv("RLHC_OMEGA_CHUNK_CTAS");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), (int64_t)per_sm * kSMs);
  note_launch(); omega_gen_kernel<<<grid, 256, 0, st>>>(seed, 0u, s, ncols, c0, Om + c0, omega_ld(m));
  return cudaGetLastError();
}

template <int NTW, bool OMEM>
static void gauss_launch(dim3 grid, const double* A, int64_t lda, int64_t rows, int n, int64_t row0, int s,
                         uint64_t seed, uint32_t stream_id, int64_t rps, double* part, const double* Om,
                         int64_t ldom, cudaStream_t st) {
  static DevFlags attr;  // per device and instantiation
  smem_attr(attr, gauss_sketch_kernel<NTW, OMEM>, (int)sizeof(GaussSmem<NTW, OMEM>));
  gauss_sketch_kernel<NTW, OMEM><<<grid, 64 * NTW, sizeof(GaussSmem<NTW, OMEM>), st>>>(
      A, lda, rows, n, row0, s, seed, stream_id, rps, part, Om, ldom);
}

cudaError_t launch_sketch_gauss(const double* A, int64_t lda, int64_t rows, int n, int64_t row0, int s, uint64_t seed,
                                uint32_t stream_id, double* part, double* out, cudaStream_t st, const double* Om) {
  GaussGeom gg = gauss_geom(rows, n, s);
  dim3 grid(gg.ti * gg.tj, gg.nsplit);
  const int64_t ldom = omega_ld(rows);
  note_launch();
  if (gg.nt == 64) {
    if (Om) gauss_launch<2, true>(grid, A, lda, rows, n, row0, s, seed, stream_id, gg.rows_per_split, part, Om, ldom, st);
    else gauss_launch<2, false>(grid, A, lda, rows, n, row0, s, seed, stream_id, gg.rows_per_split, part, Om, ldom, st);
  } else {
    if (Om) gauss_launch<8, true>(grid, A, lda, rows, n, row0, s, seed, stream_id, gg.rows_per_split, part, Om, ldom, st);
    else gauss_launch<8, false>(grid, A, lda, rows, n, row0, s, seed, stream_id, gg.rows_per_split, part, Om, ldom, st);
  }
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  const int64_t per_split = (int64_t)gg.ti * gg.tj * ST * gg.nt;
  note_launch(); gauss_reduce_kernel<<<(int)ceil_div<int64_t>(per_split, 32), 256, 0, st>>>(
      part, gg.nsplit, gg.ti * gg.tj, gg.tj, gg.nt, n, s, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ CountSketch
// plan: bucket[r], sign[r] (Philox stream 2), per-chunk histograms, bucket offsets,
// stable scatter of row ids into perm (ascending row id inside each bucket).
constexpr int CS_CHUNK = 8192;

struct CsPlan {
  int32_t* bucket;  // rows
  int8_t* sign;     // rows
  int32_t* perm;    // rows
  int32_t* hist;    // nchunks * s1 (becomes per-(chunk,bucket) base offsets)
  int32_t* start;   // s1 + 1
};
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
static CsPlan carve_plan(void* ws, int64_t rows, int s1) {
  char* p = (char*)ws;
  CsPlan pl;
  int64_t nch = ceil_div<int64_t>(rows, CS_CHUNK);
  pl.bucket = (int32_t*)p; p += align256(rows * 4);
  pl.sign = (int8_t*)p; p += align256(rows);
  pl.perm = (int32_t*)p; p += align256(rows * 4);
  pl.hist = (int32_t*)p; p += align256((size_t)nch * s1 * 4);
  pl.start = (int32_t*)p; p += align256((size_t)(s1 + 1) * 4);
  return pl;
}
size_t cs_plan_bytes(int64_t rows, int s1) {
  int64_t nch = ceil_div<int64_t>(rows, CS_CHUNK);
  return align256(rows * 4) + align256(rows) + align256(rows * 4) + align256((size_t)nch * s1 * 4) +
         align256((size_t)(s1 + 1) * 4);
}

__global__ void cs_hash_hist_kernel(int64_t rows, int64_t row0, int s1, uint64_t seed, int32_t* __restrict__ bucket,
                                    int8_t* __restrict__ sign, int32_t* __restrict__ hist) {
  extern __shared__ int h[];
  for (int b = threadIdx.x; b < s1; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * CS_CHUNK;
  for (int64_t r = c0 + threadIdx.x; r < std::min<int64_t>(rows, c0 + CS_CHUNK); r += blockDim.x) {
    int b, sg;
    cs_hash(seed, (uint64_t)(row0 + r), (uint32_t)s1, &b, &sg);
    bucket[r] = b;
    sign[r] = (int8_t)sg;
    atomicAdd(&h[b], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < s1; b += blockDim.x) hist[(int64_t)blockIdx.x * s1 + b] = h[b];
}

// per bucket: running sum over chunks -> per-(chunk, bucket) offset relative to the bucket start
__global__ void cs_bucket_totals_kernel(int nch, int s1, int32_t* __restrict__ hist, int32_t* __restrict__ start) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= s1) return;
  int run = 0;
  for (int c = 0; c < nch; c++) {
    int v = hist[(int64_t)c * s1 + b];
    hist[(int64_t)c * s1 + b] = run;
    run += v;
  }
  start[b + 1] = run;  // totals; scanned below
}

__global__ void cs_scan_kernel(int s1, int32_t* __restrict__ start) {
  // single CTA exclusive scan of totals in start[1..s1] -> start[0..s1]
  __shared__ int part[1024];
  const int per = ceil_div(s1, (int)blockDim.x);
  int b0 = threadIdx.x * per, b1 = min(s1, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; b++) sum += start[b + 1];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int q = 0; q < (int)blockDim.x; q++) { int v = part[q]; part[q] = run; run += v; }
  }
  __syncthreads();
  int run = part[threadIdx.x];
  // totals are overwritten in place with inclusive prefixes: start[b] = offset of bucket b
  for (int b = b0; b < b1; b++) { run += start[b + 1]; start[b + 1] = run; }
  __syncthreads();
  if (threadIdx.x == 0) start[0] = 0;
}

// one warp per chunk, 32 rows at a time in ascending order: stable ranks via match_any
__global__ void cs_scatter_kernel(int64_t rows, int s1, const int32_t* __restrict__ bucket,
                                  const int32_t* __restrict__ hist, const int32_t* __restrict__ start,
                                  int32_t* __restrict__ perm) {
  extern __shared__ int cnt[];
  const int lane = threadIdx.x;
  for (int b = lane; b < s1; b += 32) cnt[b] = hist[(int64_t)blockIdx.x * s1 + b] + start[b];
  __syncwarp();
  const int64_t c0 = (int64_t)blockIdx.x * CS_CHUNK, c1 = std::min<int64_t>(rows, c0 + CS_CHUNK);
  for (int64_t base = c0; base < c1; base += 32) {
    int64_t r = base + lane;
    bool ok = r < c1;
    int b = ok ? bucket[r] : -1 - lane;
    unsigned mask = __match_any_sync(0xffffffffu, b);
    int rank = __popc(mask & ((1u << lane) - 1));
    int pos = ok ? cnt[b] + rank : 0;
    __syncwarp();
    if (ok) {
      perm[pos] = (int32_t)r;
      if (rank == 0) cnt[b] += __popc(mask);
    }
    __syncwarp();
  }
}

// out[b, :] = sum over the bucket's rows (ascending) of sign * A[row, :]: one warp per
// (bucket, 32-column slice), lane = column.  The loads of 8 rows (perm, sign, values) are
// issued before their 8 additions, which stay in ascending row order (bit-exact sums).
__global__ void __launch_bounds__(256)
cs_apply_kernel(const double* __restrict__ A, int64_t lda, int n, int s1, const int32_t* __restrict__ perm,
                const int32_t* __restrict__ start, const int8_t* __restrict__ sign, double* __restrict__ out) {
  const int nslice = (n + 31) / 32;
  const int wg = blockIdx.x * (blockDim.x >> 5) + warp_id();
  const int b = wg / nslice, slice = wg - b * nslice;
  if (b >= s1) return;
  const int c = slice * 32 + lane_id();
  const bool cok = c < n;
  const int p0 = start[b], p1 = start[b + 1];
  double acc = 0.0;
  int p = p0;
  for (; p + 8 <= p1; p += 8) {
    int r[8];
    double v[8];
    bool ng[8];
#pragma unroll
    for (int u = 0; u < 8; u++) r[u] = perm[p + u];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      ng[u] = sign[r[u]] < 0;
      v[u] = cok ? A[(int64_t)r[u] * lda + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) acc = __dadd_rn(acc, ng[u] ? -v[u] : v[u]);
  }
  for (; p < p1; p++) {
    const int r = perm[p];
    const double v = cok ? A[(int64_t)r * lda + c] : 0.0;
    acc = __dadd_rn(acc, sign[r] < 0 ? -v : v);
  }
  if (cok) out[(int64_t)b * n + c] = acc;
}

// The same sums with two columns per lane (16-byte loads, 64-column slices): half the warps, each
// row's slice one 512-byte request.  Per output element the same additions in the same (bucket
// row) order, so the same bits.  A, lda: 16-byte aligned rows.
__global__ void __launch_bounds__(256)
cs_apply2_kernel(const double* __restrict__ A, int64_t lda, int n, int s1, const int32_t* __restrict__ perm,
                 const int32_t* __restrict__ start, const int8_t* __restrict__ sign, double* __restrict__ out) {
  const int nslice = (n + 63) / 64;
  const int wg = blockIdx.x * (blockDim.x >> 5) + warp_id();
  const int b = wg / nslice, slice = wg - b * nslice;
  if (b >= s1) return;
  const int c = slice * 64 + 2 * lane_id();
  const bool c0ok = c < n, c1ok = c + 1 < n;
  const int p0 = start[b], p1 = start[b + 1];
  double acc0 = 0.0, acc1 = 0.0;
  int p = p0;
  for (; p + 8 <= p1; p += 8) {
    int r[8];
    double2 v[8];
    bool ng[8];
#pragma unroll
    for (int u = 0; u < 8; u++) r[u] = perm[p + u];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      ng[u] = sign[r[u]] < 0;
      v[u] = c1ok ? *reinterpret_cast<const double2*>(A + (int64_t)r[u] * lda + c)
                  : make_double2(c0ok ? A[(int64_t)r[u] * lda + c] : 0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      acc0 = __dadd_rn(acc0, ng[u] ? -v[u].x : v[u].x);
      acc1 = __dadd_rn(acc1, ng[u] ? -v[u].y : v[u].y);
    }
  }
  for (; p < p1; p++) {
    const int r = perm[p];
    const double x = c0ok ? A[(int64_t)r * lda + c] : 0.0, y = c1ok ? A[(int64_t)r * lda + c + 1] : 0.0;
    acc0 = __dadd_rn(acc0, sign[r] < 0 ? -x : x);
    acc1 = __dadd_rn(acc1, sign[r] < 0 ? -y : y);
  }
  if (c0ok) out[(int64_t)b * n + c] = acc0;
  if (c1ok) out[(int64_t)b * n + c + 1] = acc1;
}

__global__ void copy_i32_kernel(const int32_t* a, int32_t* b, int64_t cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void copy_i8_kernel(const int8_t* a, int8_t* b, int64_t cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

cudaError_t launch_cs_plan(int64_t rows, int64_t row0, int s1, uint64_t seed, void* plan_ws, cudaStream_t st) {
  CsPlan pl = carve_plan(plan_ws, rows, s1);
  int nch = (int)ceil_div<int64_t>(rows, CS_CHUNK);
  size_t hsm = (size_t)s1 * sizeof(int);
  cudaError_t e;
  if (hsm > 48 * 1024) {
    e = cudaFuncSetAttribute(cs_hash_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    if (e) return e;
    e = cudaFuncSetAttribute(cs_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    if (e) return e;
  }
  note_launch(); cs_hash_hist_kernel<<<nch, 256, hsm, st>>>(rows, row0, s1, seed, pl.bucket, pl.sign, pl.hist);
  note_launch(); cs_bucket_totals_kernel<<<ceil_div(s1, 256), 256, 0, st>>>(nch, s1, pl.hist, pl.start);
  note_launch(); cs_scan_kernel<<<1, 1024, 0, st>>>(s1, pl.start);
  note_launch(); cs_scatter_kernel<<<nch, 32, hsm, st>>>(rows, s1, pl.bucket, pl.hist, pl.start, pl.perm);
  return cudaGetLastError();
}

cudaError_t launch_cs_apply(const double* A, int64_t lda, int64_t rows, int n, int s1, void* plan_ws, double* out,
                            cudaStream_t st) {
  CsPlan pl = carve_plan(plan_ws, rows, s1);
  static const int wide = [] { const char* e = getenv("RLHC_CS_WIDE"); return e ? atoi(e) : 1; }();
  if (wide && (lda & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    const int64_t warps = (int64_t)s1 * ((n + 63) / 64);
    note_launch();
    cs_apply2_kernel<<<(int)ceil_div<int64_t>(warps, 8), 256, 0, st>>>(A, lda, n, s1, pl.perm, pl.start, pl.sign,
                                                                       out);
    return cudaGetLastError();
  }
  const int64_t warps = (int64_t)s1 * ((n + 31) / 32);
  note_launch(); cs_apply_kernel<<<(int)ceil_div<int64_t>(warps, 8), 256, 0, st>>>(A, lda, n, s1, pl.perm, pl.start,
                                                                                    pl.sign, out);
  return cudaGetLastError();
}

cudaError_t launch_sketch_count(const double* A, int64_t lda, int64_t rows, int n, int64_t row0, int s1,
                                uint64_t seed, void* plan_ws, double* out, int32_t* bucket_out, int8_t* sign_out,
                                cudaStream_t st) {
  cudaError_t e = launch_cs_plan(rows, row0, s1, seed, plan_ws, st);
  if (e) return e;
  if ((e = launch_cs_apply(A, lda, rows, n, s1, plan_ws, out, st))) return e;
  CsPlan pl = carve_plan(plan_ws, rows, s1);
  if (bucket_out) note_launch(), copy_i32_kernel<<<256, 256, 0, st>>>(pl.bucket, bucket_out, rows);
  if (sign_out) note_launch(), copy_i8_kernel<<<256, 256, 0, st>>>(pl.sign, sign_out, rows);
  return cudaGetLastError();
}

}  // namespace rlhc
