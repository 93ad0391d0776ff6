// dist_c.cu -- row-sharded SLHC3 / SSLHC3 over NCCL, orchestrated in C (SURVEY 8(b) "_dist"
// entry points, 8(e)).  Rank r holds global rows [row0, row0 + m_local).  Per call, on the
// caller's stream, with no host synchronisation:
//   * PX = LU: per panel, the rank's leaves and local tree levels reduce to ONE tournament
//     slot (rlhc_tslu_reduce); the slots are all-gathered and every rank runs the remaining
//     levels (rlhc_tslu_combine) -> identical pivots everywhere; the pivot rows' current
//     values are assembled by an all-reduce SUM of masked per-rank copies (exact); U rows
//     follow on every rank; each rank eliminates its own rows.
//   * L of the local rows, local sketch partials indexed by global row ids -> all-reduce ->
//     replicated HouseholderQR and Y = S U.
//   * W = X Y^{-1} + local Gram -> all-reduce -> replicated Cholesky; same for V; Q = V J^{-1}
//     stays local; R = J (D Y) replicated.
// The same sequence as paper_2412_06551_b200/dist.py (which drives the stage entry points
// through torch.distributed and is checked against the oracle on CPU); every arithmetic step
// is one of the stage entry points.  NCCL is resolved at run time (dlopen "libnccl.so.2":
// whichever copy the process already has, e.g. PyTorch's), so the library has no link-time
// NCCL dependency.
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <mutex>

#include "../../include/rlhc.h"
#include "common.cuh"
#include "kernels.cuh"

namespace rlhc {
namespace {

// ---- the few NCCL entry points used (the C API is ABI-stable across 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclInt32 = 2, ncclUint64 = 5, ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0, ncclMax = 2, ncclMin = 3 } ncclRedOp_t;
typedef int ncclResult_t;

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* s) { return dlsym(h, s); };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
    n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.AllGather && n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
  });
  return n;
}

int fail(int code, const char* msg) {
  set_last_error(msg);
  return code;
}
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {
  char* p;
  size_t used = 0;
  explicit Carve(void* base) : p((char*)base) {}
  template <typename T>
  T* take(size_t count) {
    T* r = (T*)(p ? p + used : nullptr);
    used += al(count * sizeof(T));
    return r;
  }
};

int kernel_width(int panel) { return panel <= 16 ? 16 : panel <= 32 ? 32 : 64; }

// first non-OK info of the pipeline, in order (device side: no host synchronisation); the
// input check reports this rank's local element index, made global with row0 * n
__global__ void first_info_kernel(const rlhc_info_t* infos, int k, int64_t input_offset,
                                  const unsigned long long* mismatch, rlhc_info_t* out) {
  if (threadIdx.x != 0) return;
  rlhc_info_t r{0, 0, 0};
  for (int i = 0; i < k; i++)
    if (infos[i].code != 0) {
      r = infos[i];
      if (r.stage == RLHC_STAGE_INPUT) r.index += input_offset;
      break;
    }
  if (r.code == 0 && mismatch && *mismatch) r = rlhc_info_t{RLHC_ENCCL, RLHC_STAGE_COMM, (int64_t)*mismatch};
  *out = r;
}

// RLHC_DIST_CHECK: an order-sensitive 64-bit hash of `count` words (one block; debug path)
__global__ void hash_words_kernel(const unsigned long long* __restrict__ p, size_t count, unsigned long long* hmax,
                                  unsigned long long* hmin) {
  __shared__ unsigned long long red[1024];
  unsigned long long h = 0;
  for (size_t i = threadIdx.x; i < count; i += blockDim.x) {
    unsigned long long x = p[i] ^ (0x9E3779B97F4A7C15ull * (i + 1));
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    h += x;
  }
  red[threadIdx.x] = h;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *hmax = *hmin = red[0];
}
// after the max / min all-reduces: count the replicated inputs whose hashes differ
__global__ void hash_compare_kernel(const unsigned long long* hmax, const unsigned long long* hmin,
                                    unsigned long long* mismatches) {
  if (threadIdx.x == 0 && *hmax != *hmin) *mismatches += 1;
}
cudaError_t launch_hash_words(const void* p, size_t count, unsigned long long* hmax, unsigned long long* hmin,
                              cudaStream_t st) {
  note_launch();
  hash_words_kernel<<<1, 1024, 0, st>>>((const unsigned long long*)p, count, hmax, hmin);
  return cudaGetLastError();
}
cudaError_t launch_hash_compare(const unsigned long long* hmax, const unsigned long long* hmin,
                                unsigned long long* mismatches, cudaStream_t st) {
  note_launch();
  hash_compare_kernel<<<1, 32, 0, st>>>(hmax, hmin, mismatches);
  return cudaGetLastError();
}

// one info per stage call: the input check, one per panel, HQR, three solves, two Choleskys
inline int64_t max_infos(int64_t n, const rlhc_tslu_cfg& cfg) { return 1 + ceil_div<int64_t>(n, cfg.panel) + 8; }

struct DistWs {
  int64_t nslots;  // slots this rank reduces to (complete subtrees of the global tree)
  int64_t ninfos;
  unsigned long long* hash;  // RLHC_DIST_CHECK: [sum, max, min] of the replicated inputs' hashes
  int *slot_ids, *slot_cnt, *all_ids, *all_cnt, *root_ids, *root_cnt;
  double *slot_vals, *all_vals, *root_vals;
  uint8_t* chosen;
  unsigned long long* status;  // input check
  double *U, *L11, *Xp, *prow, *S, *Y, *D, *J, *N, *G, *Ls, *Lt;
  rlhc_info_t* infos;
  void* scratch;
  size_t scratch_bytes;
};

size_t scratch_need(int algo, int64_t m_local, int64_t n, int64_t s_or_s1, int64_t s2, const rlhc_tslu_cfg& cfg,
                    int nranks) {
  size_t s = 0;
  s = std::max(s, rlhc_tslu_local_workspace_size(m_local, 0, &cfg));
  s = std::max(s, rlhc_tslu_local_workspace_size(0, (int64_t)nranks * rlhc_tslu_local_slots(m_local, &cfg), &cfg));
  s = std::max(s, rlhc_tslu_panel_workspace_size(n));
  s = std::max(s, rlhc_tslu_eliminate_workspace_size(n));
  s = std::max(s, rlhc_lfactor_workspace_size(m_local, n));
  s = std::max(s, rlhc_lfactor_workspace_size(n, n));
  if (algo == RLHC_SLHC3) {
    s = std::max(s, rlhc_sketch_gauss_workspace_size(m_local, n, s_or_s1));
    s = std::max(s, rlhc_hqr_workspace_size(s_or_s1, n));
  } else {
    s = std::max(s, rlhc_sketch_count_workspace_size(m_local, n, s_or_s1));
    s = std::max(s, rlhc_sketch_gauss_workspace_size(s_or_s1, n, s2));
    s = std::max(s, rlhc_hqr_workspace_size(s2, n));
  }
  s = std::max(s, rlhc_trsm_apply_workspace_size(m_local, n));
  s = std::max(s, rlhc_cholesky_workspace_size(n));
  return s;
}

void carve_dist(Carve& c, int algo, int64_t m_local, int64_t n, int64_t s_or_s1, int64_t s2, const rlhc_tslu_cfg& cfg,
                int nranks, DistWs& d) {
  const int W = kernel_width(cfg.panel);
  const int64_t k = std::max<int64_t>(1, rlhc_tslu_local_slots(m_local, &cfg));
  d.nslots = k;
  d.ninfos = max_infos(n, cfg);
  d.hash = c.take<unsigned long long>(4);
  d.slot_ids = c.take<int>((size_t)k * W);
  d.slot_cnt = c.take<int>(k);
  d.slot_vals = c.take<double>((size_t)k * W * W);
  d.all_ids = c.take<int>((size_t)nranks * k * W);
  d.all_cnt = c.take<int>((size_t)nranks * k);
  d.all_vals = c.take<double>((size_t)nranks * k * W * W);
  d.root_ids = c.take<int>(W);
  d.root_cnt = c.take<int>(1);
  d.root_vals = c.take<double>((size_t)W * W);
  d.chosen = c.take<uint8_t>((size_t)m_local);
  d.status = c.take<unsigned long long>(4);
  double** sq[] = {&d.U, &d.L11, &d.Xp, &d.prow, &d.S, &d.Y, &d.D, &d.J, &d.N, &d.G};
  for (double** q : sq) *q = c.take<double>((size_t)n * n);
  const int64_t srows = algo == RLHC_SLHC3 ? s_or_s1 : s2;
  d.Ls = c.take<double>((size_t)srows * n);
  d.Lt = algo == RLHC_SSLHC3 ? c.take<double>((size_t)s_or_s1 * n) : nullptr;
  d.infos = c.take<rlhc_info_t>((size_t)d.ninfos);
  d.scratch_bytes = scratch_need(algo, m_local, n, s_or_s1, s2, cfg, nranks);
  d.scratch = c.take<char>(d.scratch_bytes);
}

struct DistArgs {
  int algo;
  const double* X;
  int64_t m_local, n, ldx, row0, m_global, s_or_s1, s2;
  uint64_t seed;
  rlhc_tslu_cfg cfg;
  double* Q;
  int64_t ldq;
  double* R;
  int64_t* piv;
  void* ws;
  size_t ws_bytes;
  rlhc_info_t* info;
};

}  // namespace
}  // namespace rlhc

using namespace rlhc;

struct rlhc_comm_s {
  ncclComm_t comm;
  int nranks, rank;
};

static int check_dist(const DistArgs& a, int nranks) {
  if (!a.X || !a.Q || !a.R || !a.piv || !a.ws || !a.info) return fail(RLHC_EINVAL, "null pointer argument");
  // the contract first: nothing below may divide by leaf_rows or loop on the arity before
  if (a.cfg.panel < 1 || a.cfg.panel > 64 || a.cfg.leaf_rows < 1 || a.cfg.arity < 2)
    return fail(RLHC_EINVAL, "bad tslu configuration (panel 1..64, leaf_rows >= 1, arity >= 2)");
  if (a.n < 1 || a.m_local < 1 || a.m_global < a.n) return fail(RLHC_EINVAL, "need m_global >= n >= 1, m_local >= 1");
  if (a.cfg.panel > a.n) return fail(RLHC_EINVAL, "bad tslu configuration (panel > n)");
  if (a.m_global > 0x7fffffffLL) return fail(RLHC_EINVAL, "m_global must be < 2^31 (int32 row ids)");
  if (a.ldx < a.n || a.ldq < a.n) return fail(RLHC_EINVAL, "leading dimension < n");
  if (a.m_local * nranks != a.m_global || a.row0 % a.m_local) return fail(RLHC_EINVAL, "shards must be equal");
  // equal shards of whole leaves: every rank's rows are rlhc_tslu_local_slots complete
  // subtrees of the global tree, so the pivots are the single-process contract's
  if (nranks > 1 && a.m_local % a.cfg.leaf_rows) return fail(RLHC_EINVAL, "m_local must be a multiple of leaf_rows");
  if (a.algo == RLHC_SLHC3 && (a.s_or_s1 < a.n || a.s_or_s1 > a.m_global)) return fail(RLHC_EINVAL, "need n <= s <= m");
  if (a.algo == RLHC_SSLHC3 && (a.s2 < a.n || a.s_or_s1 < a.s2 || a.s_or_s1 > a.m_global))
    return fail(RLHC_EINVAL, "need n <= s2 <= s1 <= m");
  if (((uintptr_t)a.ws) & 255) return fail(RLHC_EINVAL, "workspace must be 256-byte aligned");
  return RLHC_OK;
}

#define DTRY(x)                   \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != RLHC_OK) return rc_; \
  } while (0)
#define NTRY(x)                                                                      \
  do {                                                                               \
    ncclResult_t nr_ = (x);                                                          \
    if (nr_ != 0) return fail(RLHC_ENCCL, nccl().GetErrorString(nr_));               \
  } while (0)

static int run_dist(const DistArgs& a, rlhc_comm_t comm, cudaStream_t st) {
  Nccl& N = nccl();
  const int nr = comm ? comm->nranks : 1;
  const int64_t n = a.n, m = a.m_local;
  const int W = kernel_width(a.cfg.panel);
  Carve c(a.ws);
  DistWs d;
  carve_dist(c, a.algo, m, n, a.s_or_s1, a.s2, a.cfg, nr, d);
  if (a.ws_bytes < c.used) return fail(RLHC_EWORKSPACE, "workspace too small");
  void* sc = d.scratch;
  const size_t scb = d.scratch_bytes;
  std::function<int(const void*, size_t)> check_fn;
  auto allreduce = [&](double* p, size_t count) -> int {
    if (nr > 1) NTRY(N.AllReduce(p, p, count, ncclFloat64, ncclSum, comm->comm, st));
    return check_fn ? check_fn(p, count * sizeof(double)) : RLHC_OK;
  };
  int ninfo = 0;
  auto next_info = [&]() { return d.infos + std::min<int64_t>(ninfo++, d.ninfos - 1); };
  if (cudaMemsetAsync(d.infos, 0, (size_t)d.ninfos * sizeof(rlhc_info_t), st)) return fail(RLHC_ECUDA, "memset");
  // RLHC_DIST_CHECK=1: the replicated inputs (gathered tournament slots, all-reduced pivot
  // rows, sketch, Grams) hashed on every rank and compared through a max/min all-reduce; a
  // mismatch (e.g. a non-deterministic NVLS reduction) is reported as RLHC_ENCCL
  static const bool dcheck = [] { const char* e = getenv("RLHC_DIST_CHECK"); return e && atoi(e) != 0; }();
  if (dcheck && cudaMemsetAsync(d.hash, 0, 4 * sizeof(unsigned long long), st)) return fail(RLHC_ECUDA, "memset");
  auto check_replicated = [&](const void* p, size_t bytes) -> int {
    if (!dcheck || nr <= 1) return RLHC_OK;
    if (launch_hash_words(p, bytes / 8, d.hash + 1, d.hash + 2, st)) return fail(RLHC_ECUDA, "launch failed");
    NTRY(N.AllReduce(d.hash + 1, d.hash + 1, 1, ncclUint64, ncclMax, comm->comm, st));
    NTRY(N.AllReduce(d.hash + 2, d.hash + 2, 1, ncclUint64, ncclMin, comm->comm, st));
    if (launch_hash_compare(d.hash + 1, d.hash + 2, d.hash + 3, st)) return fail(RLHC_ECUDA, "launch failed");
    return RLHC_OK;
  };
  check_fn = check_replicated;
  const int64_t K = d.nslots;
  auto gather_slots = [&](int64_t w) -> int {  // all-gather the K slots of every rank, then the top levels
    NTRY(N.GroupStart());
    NTRY(N.AllGather(d.slot_ids, d.all_ids, (size_t)K * W, ncclInt32, comm->comm, st));
    NTRY(N.AllGather(d.slot_cnt, d.all_cnt, (size_t)K, ncclInt32, comm->comm, st));
    NTRY(N.AllGather(d.slot_vals, d.all_vals, (size_t)K * W * W, ncclFloat64, comm->comm, st));
    NTRY(N.GroupEnd());
    DTRY(check_replicated(d.all_vals, (size_t)nr * K * W * W * sizeof(double)));
    DTRY(rlhc_tslu_combine(d.all_ids, d.all_cnt, d.all_vals, nr * K, w, &a.cfg, d.root_ids, d.root_cnt, d.root_vals,
                           sc, scb, st));
    return RLHC_OK;
  };
  if (cudaMemsetAsync(d.U, 0, (size_t)n * n * sizeof(double), st)) return fail(RLHC_ECUDA, "memset");
  if (cudaMemsetAsync(d.chosen, 0, (size_t)m, st)) return fail(RLHC_ECUDA, "memset");
  // finiteness of this rank's rows (stage INPUT), first in pipeline order: folded into the
  // warp contract's Schur kernels (each reads its panel's X columns), else a pass of its own
  rlhc_info_t* input_info = next_info();
  if (launch_status_init(d.status, st)) return fail(RLHC_ECUDA, "launch failed");
  bool all_checked = true;
  // ---------------- PX = LU (P:279 / P:293), tournament over panels
  // the warp contract (leaf 128, 16-column panels): left-looking panels with the single-process
  // pipeline's arithmetic -- this rank's Schur complement of the panel into Q, the local
  // tournament (one launch), the gathered top levels, the winners' current rows from their
  // owners (all-reduced), their elimination -> U rows; L is left in Q
  const bool warp = a.cfg.leaf_rows == 128 && a.cfg.arity >= 2 && a.cfg.arity <= 8 && a.cfg.panel == 16 && n > 16;
  for (int64_t p0 = 0; warp && p0 < n; p0 += a.cfg.panel) {
    const int64_t w = std::min<int64_t>(a.cfg.panel, n - p0);
    bool checked = false;
    DTRY(tslw_schur_reduce_to_impl(a.X, m, n, a.ldx, a.Q, a.ldq, a.row0, p0, d.U, p0 > 0 ? d.chosen : nullptr,
                                   &a.cfg, nr > 1 ? K : 1, d.slot_ids, d.slot_cnt, d.slot_vals, d.status, &checked,
                                   sc, scb, st));
    all_checked = all_checked && checked;
    const int* root = d.slot_ids;
    if (nr > 1) {
      DTRY(gather_slots(w));
      root = d.root_ids;
    }
    DTRY(rlhc_tslw_owned_rows(a.X, a.ldx, a.Q, a.ldq, m, a.row0, root, w, p0, n, d.U, d.prow, st));
    DTRY(allreduce(d.prow, (size_t)w * (n - p0)));
    DTRY(rlhc_tslu_panel_factor_rows(d.prow, root, p0, w, n, a.row0, m, d.U, a.piv, d.chosen, sc, scb, next_info(),
                                     st));
  }
  if (warp) DTRY(rlhc_tslw_finish(a.Q, a.ldq, m, a.row0, n, d.U, a.piv, st));
  if (!warp || !all_checked) {
    if (launch_check_finite(a.X, m, (int)n, a.ldx, d.status, st)) return fail(RLHC_ECUDA, "launch failed");
  }
  if (launch_status_finish(d.status, input_info, st)) return fail(RLHC_ECUDA, "launch failed");
  for (int64_t p0 = 0; !warp && p0 < n; p0 += a.cfg.panel) {
    const int64_t w = std::min<int64_t>(a.cfg.panel, n - p0);
    const double* src = p0 == 0 ? a.X : a.Q;
    const int64_t lds = p0 == 0 ? a.ldx : a.ldq;
    DTRY(rlhc_tslu_reduce_to(src, lds, m, a.row0, p0, w, p0 > 0 ? d.chosen : nullptr, &a.cfg, nr > 1 ? K : 1,
                             d.slot_ids, d.slot_cnt, d.slot_vals, sc, scb, st));
    const int* root = d.slot_ids;
    if (nr > 1) {
      DTRY(gather_slots(w));
      root = d.root_ids;
    }
    DTRY(rlhc_owned_rows(src, lds, m, a.row0, root, nullptr, w, p0, n - p0, d.prow, st));
    DTRY(allreduce(d.prow, (size_t)w * (n - p0)));
    DTRY(rlhc_tslu_panel_factor_rows(d.prow, root, p0, w, n, a.row0, m, d.U, a.piv, d.chosen, sc, scb, next_info(),
                                     st));
    if (p0 + w < n) DTRY(rlhc_tslu_eliminate(src, lds, m, p0, w, n, d.U, a.Q, a.ldq, sc, scb, st));
  }
  if (!warp) {
    DTRY(rlhc_owned_rows(a.X, a.ldx, m, a.row0, nullptr, a.piv, n, 0, n, d.Xp, st));
    DTRY(allreduce(d.Xp, (size_t)n * n));
    DTRY(rlhc_l11(d.Xp, n, d.U, d.L11, sc, scb, st));
    DTRY(rlhc_lfactor(a.X, m, n, a.ldx, a.row0, d.U, d.L11, a.piv, a.Q, a.ldq, sc, scb, st));
  }
  // ---------------- sketch of L (P:280 / P:294): local partials, all-reduced
  int64_t srows;
  if (a.algo == RLHC_SLHC3) {
    srows = a.s_or_s1;
    DTRY(rlhc_sketch_gauss(a.Q, m, n, a.ldq, a.row0, srows, a.seed, 0, d.Ls, sc, scb, st));
    DTRY(allreduce(d.Ls, (size_t)srows * n));
  } else {
    srows = a.s2;
    DTRY(rlhc_sketch_count(a.Q, m, n, a.ldq, a.row0, a.s_or_s1, a.seed, d.Lt, nullptr, nullptr, sc, scb, st));
    DTRY(allreduce(d.Lt, (size_t)a.s_or_s1 * n));
    DTRY(rlhc_sketch_gauss(d.Lt, a.s_or_s1, n, n, 0, srows, a.seed, 1, d.Ls, sc, scb, st));
  }
  // ---------------- [H, S] = HouseholderQR(L_s) (R#7), Y = S U
  DTRY(rlhc_hqr_r(d.Ls, srows, n, n, d.U, d.S, sc, scb, next_info(), st));
  DTRY(rlhc_trmm_upper(d.S, d.U, n, d.Y, st));
  // ---------------- W = X Y^{-1} (+ G1), CholeskyQR2, R = J (D Y)
  DTRY(rlhc_trsm_apply(a.X, m, n, a.ldx, d.Y, RLHC_SUBST, a.Q, a.ldq, d.G, sc, scb, next_info(), st));
  DTRY(allreduce(d.G, (size_t)n * n));
  DTRY(rlhc_cholesky_ws(d.G, n, d.D, RLHC_STAGE_CHOL1, sc, scb, next_info(), st));
  // the CholeskyQR passes as on one GPU (run_algo): n > 64 the explicit inverse and the in-place
  // triangular product (R#9: kappa(D), kappa(J) <= ~7)
  const int cq_mode = n > 64 ? RLHC_INV_GEMM : RLHC_SUBST;
  DTRY(rlhc_trsm_apply(a.Q, m, n, a.ldq, d.D, cq_mode, a.Q, a.ldq, d.G, sc, scb, next_info(), st));
  DTRY(allreduce(d.G, (size_t)n * n));
  DTRY(rlhc_cholesky_ws(d.G, n, d.J, RLHC_STAGE_CHOL2, sc, scb, next_info(), st));
  DTRY(rlhc_trsm_apply(a.Q, m, n, a.ldq, d.J, cq_mode, a.Q, a.ldq, nullptr, sc, scb, next_info(), st));
  DTRY(rlhc_trmm_upper(d.D, d.Y, n, d.N, st));
  DTRY(rlhc_trmm_upper(d.J, d.N, n, a.R, st));
  note_launch();
  first_info_kernel<<<1, 32, 0, st>>>(d.infos, (int)std::min<int64_t>(ninfo, d.ninfos), a.row0 * n,
                                      dcheck ? d.hash + 3 : nullptr, a.info);
  if (cudaGetLastError()) return fail(RLHC_ECUDA, "launch failed");
  return RLHC_OK;
}

extern "C" {

int rlhc_comm_unique_id(void* id_out) {
  if (!id_out) return fail(RLHC_EINVAL, "null pointer argument");
  Nccl& N = nccl();
  if (!N.ok) return fail(RLHC_ENCCL, "libnccl.so.2 not found");
  NTRY(N.GetUniqueId((ncclUniqueId*)id_out));
  return RLHC_OK;
}

int rlhc_comm_init(rlhc_comm_t* comm, int nranks, int rank, const void* id) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(RLHC_EINVAL, "bad arguments");
  Nccl& N = nccl();
  if (!N.ok) return fail(RLHC_ENCCL, "libnccl.so.2 not found");
  rlhc_comm_s* c = new rlhc_comm_s{nullptr, nranks, rank};
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = N.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != 0) {
    delete c;
    return fail(RLHC_ENCCL, N.GetErrorString(r));
  }
  *comm = c;
  return RLHC_OK;
}

int rlhc_comm_destroy(rlhc_comm_t comm) {
  if (!comm) return RLHC_OK;
  Nccl& N = nccl();
  ncclResult_t r = N.CommDestroy(comm->comm);
  delete comm;
  return r == 0 ? RLHC_OK : fail(RLHC_ENCCL, N.GetErrorString(r));
}

size_t rlhc_dist_workspace_size(int algo, int64_t m_local, int64_t n, int64_t s_or_s1, int64_t s2,
                                const rlhc_tslu_cfg* cfg, int nranks) {
  if (!cfg || n < 1 || m_local < 1 || nranks < 1) return 0;
  if (cfg->panel < 1 || cfg->panel > 64 || cfg->leaf_rows < 1 || cfg->arity < 2) return 0;
  if (algo != RLHC_SLHC3 && algo != RLHC_SSLHC3) return 0;
  Carve c(nullptr);
  DistWs d;
  carve_dist(c, algo, m_local, n, s_or_s1, s2, *cfg, nranks, d);
  return c.used;
}

int rlhc_slhc3_dist(const double* X, int64_t m_local, int64_t n, int64_t ldx, int64_t row0, int64_t m_global,
                    int64_t s, uint64_t seed, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq, double* R,
                    int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_comm_t comm,
                    rlhc_stream_t stream) {
  if (!cfg) return fail(RLHC_EINVAL, "null tslu configuration");
  DistArgs a{RLHC_SLHC3, X, m_local, n, ldx, row0, m_global, s, 0, seed, *cfg, Q, ldq, R, piv, ws, ws_bytes, info};
  const int nr = comm ? comm->nranks : 1;
  int rc = check_dist(a, nr);
  if (rc) return rc;
  return run_dist(a, comm, (cudaStream_t)stream);
}

int rlhc_sslhc3_dist(const double* X, int64_t m_local, int64_t n, int64_t ldx, int64_t row0, int64_t m_global,
                     int64_t s1, int64_t s2, uint64_t seed, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq,
                     double* R, int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_comm_t comm,
                     rlhc_stream_t stream) {
  if (!cfg) return fail(RLHC_EINVAL, "null tslu configuration");
  DistArgs a{RLHC_SSLHC3, X, m_local, n, ldx, row0, m_global, s1, s2, seed, *cfg, Q, ldq, R, piv, ws, ws_bytes, info};
  const int nr = comm ? comm->nranks : 1;
  int rc = check_dist(a, nr);
  if (rc) return rc;
  return run_dist(a, comm, (cudaStream_t)stream);
}

}  // extern "C"
