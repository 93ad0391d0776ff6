// rlhc.cu -- the C ABI (include/rlhc.h): argument checks, workspace carving and the
// stream-ordered pipelines of SLHC3 and SSLHC3.  No host
// synchronisation and no allocation inside a call; every stage is a kernel of this
// library (tslu.cu, rows.cu, sketch.cu, small.cu).
#include <array>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace rlhc;

static thread_local std::string g_last_error;
namespace rlhc {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace rlhc

static int fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
#define CUDA_TRY(x)                                                         \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      g_last_error = std::string(#x) + ": " + cudaGetErrorString(e_);       \
      return RLHC_ECUDA;                                                    \
    }                                                                       \
  } while (0)

namespace {

// ---------------------------------------------------------------- stage timing
constexpr int kStages = RLHC_NUM_TIMED_STAGES;
const char* kStageNames[kStages] = {"check_finite", "tslu",  "lfactor", "sketch", "hqr_y", "solve_w", "gram1",
                                    "chol1",        "solve_v", "gram2",  "chol2",  "solve_q", "r_finish"};
using MarkSet = std::array<cudaEvent_t, kStages + 1>;
struct StageProf {
  std::mutex mu;
  bool enabled = false;
  std::vector<MarkSet> pending, pool;
} g_prof;

struct Marks {
  MarkSet ev{};
  bool on = false;
  cudaStream_t st = nullptr;
  void mark(int k) {
    if (on) cudaEventRecord(ev[k], st);
  }
};

Marks prof_begin(cudaStream_t st) {
  Marks m;
  std::lock_guard<std::mutex> g(g_prof.mu);
  if (!g_prof.enabled) return m;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return m;
  if (!g_prof.pool.empty()) {
    m.ev = g_prof.pool.back();
    g_prof.pool.pop_back();
  } else {
    for (auto& e : m.ev)
      if (cudaEventCreate(&e) != cudaSuccess) return Marks{};
  }
  m.on = true;
  m.st = st;
  return m;
}
void prof_end(Marks& m) {
  if (!m.on) return;
  std::lock_guard<std::mutex> g(g_prof.mu);
  g_prof.pending.push_back(m.ev);
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

int kernel_width(int panel) { return panel <= 16 ? 16 : (panel <= 32 ? 32 : 64); }

bool cfg_ok(const rlhc_tslu_cfg& c, int64_t m, int64_t n) {
  if (c.panel < 1 || c.panel > 64 || c.panel > n) return false;
  if (tslw_cfg(c, m, n)) return true;
  int W = kernel_width(c.panel);
  if (c.leaf_rows < 1 || c.leaf_rows > select_rows(W)) return false;
  if (c.arity < 2 || (int64_t)c.arity * c.panel > select_rows(W)) return false;
  return true;
}

struct Carver {
  char* p;
  size_t used = 0;
  explicit Carver(void* base) : p((char*)base) {}
  template <typename T>
  T* take(size_t count) {
    T* r = (T*)(p ? p + used : nullptr);
    used += al(count * sizeof(T));
    return r;
  }
};

struct TsluWs {
  unsigned long long* status;
  uint8_t* chosen;
  int* ids[2];
  int* cnt[2];
  double* vals[2];
  double* rd;
  double* lw;
  double* Xp;
  void* gepp;  // exact GEPP mode: the panel's working copy
  double* bpack;  // the grouped LU's bulk products (tsgemm.cu packed B)
};

void carve_tslu(Carver& c, int64_t rows, int64_t n, const rlhc_tslu_cfg& cfg, TsluWs& t) {
  int W = kernel_width(cfg.panel);
  int64_t nleaves = ceil_div<int64_t>(rows, cfg.leaf_rows);
  for (int b = 0; b < 2; b++) {
    t.ids[b] = c.take<int>((size_t)nleaves * W);
    t.cnt[b] = c.take<int>((size_t)2 * nleaves + 64);  // tslw: packed counts + arrival counters
    t.vals[b] = c.take<double>((size_t)nleaves * W * W);
  }
  t.chosen = c.take<uint8_t>((size_t)rows);
  t.rd = c.take<double>((size_t)n);
  t.lw = c.take<double>((size_t)kTslwPanel * kTslwPanel);
  t.gepp = tslg_cfg(cfg, rows, n) ? (void*)c.take<char>(tslg_ws_bytes(rows)) : nullptr;
  t.bpack = c.take<double>(ts_gemm_pack_bytes((int)n, kTslwGroup) / sizeof(double));
  t.Xp = c.take<double>((size_t)n * n);
}

// PX = LU on rows x n (global ids row0..): piv, U, L11; the trailing matrix of later
// panels lives in `tw` (rows x n, ldt).  Returns RLHC_OK or RLHC_ECUDA.
int run_tslu(const double* X, int64_t rows, int64_t n, int64_t ldx, int64_t row0, const rlhc_tslu_cfg& cfg,
             TsluWs& t, double* tw, int64_t ldtw, int64_t* piv, double* U, double* L11, cudaStream_t st,
             bool check_input = false, const TslwPanelHook* hook = nullptr) {
  if (tslw_cfg(cfg, rows, n)) {  // warp tournament (or exact GEPP); L (original row order) lands in tw
    CUDA_TRY(run_tslw(X, ldx, rows, row0, (int)n, cfg.arity, tw, ldtw, piv, U, L11, t.rd, t.lw, t.chosen, t.ids,
                      t.cnt, t.vals, t.status, check_input, st, t.gepp, t.bpack, hook));
    return RLHC_OK;
  }
  const int W = kernel_width(cfg.panel);
  const int nleaves = (int)ceil_div<int64_t>(rows, cfg.leaf_rows);
  const bool panels = cfg.panel < n;
  if (panels) CUDA_TRY(cudaMemsetAsync(t.chosen, 0, (size_t)rows, st));
  CUDA_TRY(cudaMemsetAsync(U, 0, (size_t)n * n * sizeof(double), st));  // strict lower part of U is 0
  // single panel, single process: the root node's GEPP already computes U, the L11
  // multipliers and 1/diag(U) (same fma chains as the panel elimination), so it emits them
  const bool root_emit = !panels && row0 == 0;
  RootOut ro{U, piv, L11, t.rd, t.status, (int)n};
  for (int64_t p0 = 0; p0 < n; p0 += cfg.panel) {
    const int w = (int)std::min<int64_t>(cfg.panel, n - p0);
    const double* src = (p0 == 0) ? X : tw;
    const int64_t lds = (p0 == 0) ? ldx : ldtw;
    // slots carry ids only: every node reads its candidates' rows from src by global id
    const RowSrc rsrc{src, lds, row0, (int)p0};
    CUDA_TRY(launch_tslu_leaf(W, cfg.leaf_rows, src, lds, rows, row0, (int)p0, w, panels && p0 > 0 ? t.chosen : nullptr, t.ids[0],
                              t.cnt[0], nullptr, st, root_emit && nleaves == 1 ? &ro : nullptr,
                              check_input && !panels ? t.status : nullptr));
    int cur = 0, nslots = nleaves;
    while (nslots > 1) {
      const int nout = (int)ceil_div<int64_t>(nslots, cfg.arity);
      CUDA_TRY(launch_tslu_node(W, t.ids[cur], t.cnt[cur], nullptr, nslots, cfg.arity, w, t.ids[cur ^ 1],
                                t.cnt[cur ^ 1], nullptr, st, root_emit && nout == 1 ? &ro : nullptr, &rsrc));
      nslots = nout;
      cur ^= 1;
    }
    if (root_emit) return RLHC_OK;
    CUDA_TRY(launch_tslu_panel_factor(src, lds, rows, row0, (int)p0, w, (int)n, t.ids[cur], t.cnt[cur], U, piv,
                                      panels ? t.chosen : nullptr, nullptr, t.status, st));
    CUDA_TRY(launch_rdiag(U + p0 * n + p0, w, n + 0, t.rd + p0, RLHC_STAGE_LU, t.status, st));
    if (p0 + w < n) {
      // eliminate every row with this panel's pivots: multipliers (substitution over
      // the panel) and the fma-chain update of the trailing columns
      CUDA_TRY(launch_trsm_rows(src + p0, lds, rows, (int)(n - p0), w, U + p0 * n + p0, n, t.rd + p0, tw + p0, ldtw,
                                nullptr, nullptr, 0, st));
    }
  }
  // L11: the pivot rows' X rows run through the same substitution, unit diagonal
  CUDA_TRY(launch_gather_rows(X, ldx, piv, row0, (int)n, (int)n, t.Xp, n, st));
  CUDA_TRY(launch_trsm_rows(t.Xp, n, n, (int)n, (int)n, U, n, t.rd, L11, n, nullptr, nullptr, 0, st));
  CUDA_TRY(launch_l11_fixup(L11, (int)n, st));
  return RLHC_OK;
}

struct AlgoWs {
  TsluWs t;
  int* pivpos;
  double *U, *L11, *S, *Y, *G, *D, *Di, *J, *Ji, *N, *rdY, *Tinv, *bpack;
  double *Lt, *Ls, *part, *work;
  void* plan;
  double* Om;  // the stored Gaussian sketch (nullptr: generated inside the sketch kernel)
};

// Omega (and the CountSketch plan) depend only on the seed and the sizes: they are produced
// on a side stream forked at the start of the call, overlapping the latency-bound TSLU, and
// joined before the sketch.  Bounded so that huge sketches keep the in-kernel generator.
constexpr size_t kOmegaStoreMax = size_t(4) << 30;
// SLHC3 stores Omega only for n > 256, where the in-kernel generator would redo it for
// every 256-column tile; below that the side-stream generator costs the TSLU more than it
// saves the sketch (cfg2: TSLU +45 us, sketch -35 us).  RLHC_OMEGA_STORE=0/1 overrides
// (measurement knob).
// SLHC3 with 16 < n <= 256 under the warp-tournament contract generates Omega in one chunk per
// panel on a low-priority side stream, each chunk released when its panel's Schur kernel is
// done, so that it runs in the SMs the panel's tournament leaves idle (RLHC_OMEGA_CHUNKS=0:
// the in-kernel generator instead).
static bool omega_chunked(int algo, int64_t m, int64_t n, const rlhc_tslu_cfg& cfg) {
  static const int on = [] {
    const char* e = getenv("RLHC_OMEGA_CHUNKS");
    return e ? atoi(e) : 1;
  }();
  return on && algo == RLHC_SLHC3 && n > 16 && n <= 256 && tslw_cfg(cfg, m, n);  // >= 2 panels
}
static size_t omega_store_bytes(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2,
                                const rlhc_tslu_cfg& cfg) {
  static const int force = [] {
    const char* e = getenv("RLHC_OMEGA_STORE");
    return e ? atoi(e) : -1;
  }();
  const bool want = force >= 0 ? force != 0 : (algo == RLHC_SSLHC3 || n > 256 || omega_chunked(algo, m, n, cfg));
  const size_t b = algo == RLHC_SLHC3 ? omega_bytes(s_or_s1, m) : omega_bytes(s2, s_or_s1);
  return want && b <= kOmegaStoreMax ? b : 0;
}

// one non-blocking side stream and a fork/join event pair per host thread and device
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static cudaError_t side_stream(SideStream** out) {
  static thread_local std::array<SideStream, 64> per_dev;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  SideStream& ss = per_dev[dev];
  if (!ss.s) {
    // lowest priority: its work is off the critical path, pending CTAs of the main stream
    // are scheduled first
    int least = 0, greatest = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&least, &greatest))) return e;
    if ((e = cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, least))) return e;
    if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming))) return e;
  }
  *out = &ss;
  return cudaSuccess;
}
// joins the side stream back into `st` on every exit path (a capture must not end forked)
struct SideJoin {
  cudaStream_t st = nullptr;
  SideStream* ss = nullptr;
  cudaError_t join() {
    if (!ss) return cudaSuccess;
    SideStream* p = ss;
    ss = nullptr;
    return cudaStreamWaitEvent(st, p->join, 0);
  }
  ~SideJoin() { join(); }
};

void carve_algo(Carver& c, int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2, const rlhc_tslu_cfg& cfg,
                AlgoWs& a) {
  a.t.status = c.take<unsigned long long>(4);
  carve_tslu(c, m, n, cfg, a.t);
  a.pivpos = c.take<int>((size_t)m);
  double** sq[] = {&a.U, &a.L11, &a.S, &a.Y, &a.G, &a.D, &a.Di, &a.J, &a.Ji, &a.N, &a.Tinv};
  for (double** q : sq) *q = c.take<double>((size_t)n * n);
  a.rdY = c.take<double>((size_t)n);
  a.bpack = c.take<double>(ts_gemm_pack_bytes((int)n, (int)n) / sizeof(double));
  const int64_t srows = algo == RLHC_SLHC3 ? s_or_s1 : s2;
  a.Ls = c.take<double>((size_t)srows * n);
  a.Lt = algo == RLHC_SSLHC3 ? c.take<double>((size_t)s_or_s1 * n) : nullptr;
  size_t part = std::max(gram_partials_bytes(m, (int)n), rowsolve_partials_bytes(m, (int)n));
  part = std::max(part, subst_ms_partials_bytes(m, (int)n));
  part = std::max(part, algo == RLHC_SLHC3 ? gauss_partials_bytes(m, (int)n, (int)s_or_s1)
                                           : gauss_partials_bytes(s_or_s1, (int)n, (int)s2));
  a.part = c.take<double>(part / sizeof(double) + 1);
  size_t work = std::max(hqr_ws_bytes((int)srows, (int)n), chol_ws_bytes((int)n));
  a.work = c.take<double>(work / sizeof(double) + 1);
  a.plan = algo == RLHC_SSLHC3 ? (void*)c.take<char>(cs_plan_bytes(m, (int)s_or_s1)) : nullptr;
  const size_t ob = omega_store_bytes(algo, m, n, s_or_s1, s2, cfg);
  a.Om = ob ? c.take<double>(ob / sizeof(double)) : nullptr;
}

int run_algo(int algo, const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s_or_s1, int64_t s2, uint64_t seed,
             const rlhc_tslu_cfg& cfg, double* Q, int64_t ldq, double* R, int64_t* piv, AlgoWs& a, rlhc_info_t* info,
             cudaStream_t st) {
  const int ni = (int)n;
  unsigned long long* status = a.t.status;
  Marks mk = prof_begin(st);
  mk.mark(0);
  CUDA_TRY(launch_status_init(status, st));
  // side stream: Omega (SLHC3: s x m; SSLHC3: s2 x s1) and the CountSketch plan
  SideJoin side;
  const bool chunked = a.Om && omega_chunked(algo, m, n, cfg);
  struct OmegaChunks {
    SideStream* ss;
    uint64_t seed;
    int s;
    int64_t m;
    double* Om;
  } oc{nullptr, seed, (int)s_or_s1, m, a.Om};
  TslwPanelHook hook{[](void* ctx, int panel, int npanels, cudaStream_t st0) -> cudaError_t {
                       OmegaChunks& o = *static_cast<OmegaChunks*>(ctx);
                       const int64_t c0 = o.m * panel / npanels, c1 = o.m * (panel + 1) / npanels;
                       cudaError_t e = cudaEventRecord(o.ss->fork, st0);
                       if (!e) e = cudaStreamWaitEvent(o.ss->s, o.ss->fork, 0);
                       if (!e) e = launch_omega_gen_cols(o.seed, o.s, o.m, c0, c1 - c0, o.Om, o.ss->s);
                       if (!e) e = cudaEventRecord(o.ss->join, o.ss->s);
                       return e;
                     },
                     &oc};
  if (chunked) {
    CUDA_TRY(side_stream(&oc.ss));
    side.st = st;
    side.ss = oc.ss;
  } else if (a.Om) {
    SideStream* ss = nullptr;
    CUDA_TRY(side_stream(&ss));
    CUDA_TRY(cudaEventRecord(ss->fork, st));
    CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    side.st = st;
    side.ss = ss;
    if (algo == RLHC_SLHC3) {
      CUDA_TRY(launch_omega_gen(seed, 0u, (int)s_or_s1, m, 0, a.Om, ss->s));
    } else {
      CUDA_TRY(launch_cs_plan(m, 0, (int)s_or_s1, seed, a.plan, ss->s));
      CUDA_TRY(launch_omega_gen(seed, 1u, (int)s2, s_or_s1, 0, a.Om, ss->s));
    }
    CUDA_TRY(cudaEventRecord(ss->join, ss->s));
  }
  // input check: a pass of its own, or (one panel) folded into the TSLU leaves' read of X
  const bool fold_check = cfg.panel >= n || tslw_cfg(cfg, m, n);
  if (!fold_check) CUDA_TRY(launch_check_finite(X, m, ni, ldx, status, st));
  mk.mark(1);
  // PX = LU (P:279 / P:293); the Q buffer holds the trailing matrix of later panels
  int rc = run_tslu(X, m, n, ldx, 0, cfg, a.t, Q, ldq, piv, a.U, a.L11, st, fold_check, chunked ? &hook : nullptr);
  if (rc) return rc;
  const bool l_done = tslw_cfg(cfg, m, n);  // the warp tournament leaves L in the Q buffer
  if (!l_done) {
    CUDA_TRY(launch_fill_i32(a.pivpos, m, -1, st));
    CUDA_TRY(launch_pivpos(piv, ni, 0, m, a.pivpos, st));
  }
  mk.mark(2);
  // one streaming pass: out = A T^{-1} (substitution) [+ G = out^T out fused]
  // ms: the oracle's op sequence (DESIGN.md R#O9) for solves with an ill-conditioned T (W = X Y^{-1});
  // the CholeskyQR passes (kappa(D), kappa(J) <= ~7) keep the faster fma chain
  // gmark: stage marker between the solve and a separate Gram (-1: none; with a fused Gram the
  // Gram stage is empty)
  auto solve_pass = [&](const double* A, int64_t lda, const double* T, const double* rd, const int* pp,
                        const double* l11, double* G, bool ms = false, int gmark = -1) -> int {
    if (ms && !pp && subst_ms_ok(ni)) {  // the oracle's op sequence (DESIGN.md R#O9), then the Gram
      CUDA_TRY(launch_subst_ms(A, lda, m, ni, T, n, Q, ldq, a.part, G, st));
      if (gmark >= 0) mk.mark(gmark);
    } else if (ms && !pp && subst_wide_ok(ni)) {  // the same sequence for n > 64 (subst.cu), then the Gram
      CUDA_TRY(launch_subst_wide(A, lda, m, ni, T, n, Q, ldq, st));
      if (gmark >= 0) mk.mark(gmark);
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    } else if (rowsolve_ok(ni)) {
      CUDA_TRY(launch_rowsolve(A, lda, m, ni, T, rd, Q, ldq, pp ? piv : nullptr, l11, a.part, G, st));
      if (gmark >= 0) mk.mark(gmark);
    } else if (!ms && !pp) {
      // a CholeskyQR pass, n > 64: T = D or J (kappa <= ~7) -> explicit inverse
      // (R#9) and the in-place triangular product on DMMA (tsgemm.cu), then the Gram
      CUDA_TRY(launch_tri_inv(T, ni, a.Tinv, st));
      CUDA_TRY(launch_ts_gemm(nullptr, 0, Q, ldq, A, lda, a.Tinv, n, m, ni, ni, true, false, a.bpack, st));
      if (gmark >= 0) mk.mark(gmark);
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    } else {
      CUDA_TRY(launch_trsm_blocked(A, lda, m, ni, ni, T, n, rd, Q, ldq, st));
      if (pp) CUDA_TRY(launch_pivot_rows(piv, ni, 0, m, l11, Q, ldq, st));
      if (gmark >= 0) mk.mark(gmark);
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    }
    return RLHC_OK;
  };
  // L in original row order (R#2), into the Q buffer
  if (!l_done && (rc = solve_pass(X, ldx, a.U, a.t.rd, a.pivpos, a.L11, nullptr))) return rc;
  mk.mark(3);
  int64_t srows;
  CUDA_TRY(side.join());
  if (algo == RLHC_SLHC3) {  // L_s = Omega L
    srows = s_or_s1;
    CUDA_TRY(launch_sketch_gauss(Q, ldq, m, ni, 0, (int)srows, seed, 0u, a.part, a.Ls, st, a.Om));
  } else {                   // L_t = Omega_1 L, L_ss = Omega_2 L_t
    srows = s2;
    if (a.Om) CUDA_TRY(launch_cs_apply(Q, ldq, m, ni, (int)s_or_s1, a.plan, a.Lt, st));
    else CUDA_TRY(launch_sketch_count(Q, ldq, m, ni, 0, (int)s_or_s1, seed, a.plan, a.Lt, nullptr, nullptr, st));
    CUDA_TRY(launch_sketch_gauss(a.Lt, n, s_or_s1, ni, 0, (int)s2, seed, 1u, a.part, a.Ls, st, a.Om));
  }
  mk.mark(4);
  // [H, S] = HouseholderQR(L_s), sign(S_kk) = sign(U_kk) (R#7); Y = S U
  CUDA_TRY(launch_hqr(a.Ls, (int)srows, ni, n, a.U, a.S, a.work, status, st));
  CUDA_TRY(launch_trmm_uu(a.S, a.U, ni, a.Y, st));
  CUDA_TRY(launch_rdiag(a.Y, ni, n, a.rdY, RLHC_STAGE_SOLVE_Y, status, st));
  mk.mark(5);
  // W = X Y^{-1} by substitution, fused G1 = W^T W (first Gram of CholeskyQR2)
  if ((rc = solve_pass(X, ldx, a.Y, a.rdY, nullptr, nullptr, a.G, true, 6))) return rc;
  mk.mark(7);
  // CholeskyQR2(W): D = chol(G1), V = W D^{-1} (+ G2), J = chol(G2), Q = V J^{-1}
  CUDA_TRY(launch_chol(a.G, ni, a.D, a.work, RLHC_STAGE_CHOL1, status, st, ni <= 128 ? a.Di : nullptr));
  if (ni > 128) CUDA_TRY(launch_rdiag(a.D, ni, n, a.Di, RLHC_STAGE_SOLVE_D, status, st));
  mk.mark(8);
  // NEXT-4 (n <= 64, RLHC_Q_JD=1): V = W D^{-1} is formed tile by tile only for G2 and never
  // stored (Q keeps W), and Q = W (J D)^{-1} -- 7 passes of m x n instead of 8
  static const bool q_jd = [] { const char* e = getenv("RLHC_Q_JD"); return e && atoi(e) != 0; }();
  const bool jd = q_jd && rowsolve_ok(ni);
  if (jd) {
    CUDA_TRY(launch_rowsolve(Q, ldq, m, ni, a.D, a.Di, nullptr, ldq, nullptr, nullptr, a.part, a.G, st));
    mk.mark(9);
  } else if ((rc = solve_pass(Q, ldq, a.D, a.Di, nullptr, nullptr, a.G, false, 9))) {
    return rc;
  }
  mk.mark(10);
  CUDA_TRY(launch_chol(a.G, ni, a.J, a.work, RLHC_STAGE_CHOL2, status, st, ni <= 128 ? a.Ji : nullptr));
  if (ni > 128) CUDA_TRY(launch_rdiag(a.J, ni, n, a.Ji, RLHC_STAGE_SOLVE_J, status, st));
  if (jd) {  // T = J D (S is free since Y = S U), 1/diag(T) over J's reciprocals
    CUDA_TRY(launch_trmm_uu(a.J, a.D, ni, a.S, st));
    CUDA_TRY(launch_rdiag(a.S, ni, n, a.Ji, RLHC_STAGE_SOLVE_J, status, st));
  }
  mk.mark(11);
  if ((rc = solve_pass(Q, ldq, jd ? a.S : a.J, a.Ji, nullptr, nullptr, nullptr))) return rc;
  mk.mark(12);
  // R = Z Y = J (D Y)
  CUDA_TRY(launch_trmm_uu(a.D, a.Y, ni, a.N, st));
  CUDA_TRY(launch_trmm_uu(a.J, a.N, ni, R, st));
  CUDA_TRY(launch_status_finish(status, info, st));
  mk.mark(13);
  prof_end(mk);
  return RLHC_OK;
}

// ---- the paper's comparison algorithms on the same kernels (the oracle's
// ora_cholqr2 / ora_scholqr3 / ora_luc2 / ora_rhc).  Workspace: the SSLHC3 layout with
// s1 = max(s1, n), s2 = max(s2, n) covers every method.
int run_method(int method, const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed,
               const rlhc_tslu_cfg& cfg, double* Q, int64_t ldq, double* R, int64_t* piv, AlgoWs& a, rlhc_info_t* info,
               cudaStream_t st) {
  const int ni = (int)n;
  unsigned long long* status = a.t.status;
  CUDA_TRY(launch_status_init(status, st));
  CUDA_TRY(launch_check_finite(X, m, ni, ldx, status, st));
  // out = A T^{-1} (substitution, into Q) [+ G = out^T out]
  // ms: the oracle's op sequence (DESIGN.md R#O9) for solves with an ill-conditioned T (W = X Y^{-1});
  // the CholeskyQR passes (kappa(D), kappa(J) <= ~7) keep the faster fma chain
  auto solve_pass = [&](const double* A, int64_t lda, const double* T, const double* rd, const int* pp,
                        const double* l11, double* G, bool ms = false) -> int {
    if (ms && !pp && subst_ms_ok(ni)) {  // the oracle's op sequence (DESIGN.md R#O9), then the Gram
      CUDA_TRY(launch_subst_ms(A, lda, m, ni, T, n, Q, ldq, a.part, G, st));
    } else if (ms && !pp && subst_wide_ok(ni)) {  // the same sequence for n > 64 (subst.cu), then the Gram
      CUDA_TRY(launch_subst_wide(A, lda, m, ni, T, n, Q, ldq, st));
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    } else if (rowsolve_ok(ni)) {
      CUDA_TRY(launch_rowsolve(A, lda, m, ni, T, rd, Q, ldq, pp ? piv : nullptr, l11, a.part, G, st));
    } else if (!ms && !pp) {
      // a CholeskyQR pass, n > 64: T = D or J (kappa <= ~7) -> explicit inverse
      // (R#9) and the in-place triangular product on DMMA (tsgemm.cu), then the Gram
      CUDA_TRY(launch_tri_inv(T, ni, a.Tinv, st));
      CUDA_TRY(launch_ts_gemm(nullptr, 0, Q, ldq, A, lda, a.Tinv, n, m, ni, ni, true, false, a.bpack, st));
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    } else {
      CUDA_TRY(launch_trsm_blocked(A, lda, m, ni, ni, T, n, rd, Q, ldq, st));
      if (pp) CUDA_TRY(launch_pivot_rows(piv, ni, 0, m, l11, Q, ldq, st));
      if (G) CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, G, st));
    }
    return RLHC_OK;
  };
  // T = Cholesky(G) with its 1/diag for the next substitution
  auto chol = [&](double* T, double* rd, int stage) -> int {
    CUDA_TRY(launch_chol(a.G, ni, T, a.work, stage, status, st, ni <= 128 ? rd : nullptr));
    const int solve_stage = stage == RLHC_STAGE_CHOL0 ? RLHC_STAGE_SOLVE_Y
                            : stage == RLHC_STAGE_CHOL1 ? RLHC_STAGE_SOLVE_D : RLHC_STAGE_SOLVE_J;
    if (ni > 128) CUDA_TRY(launch_rdiag(T, ni, n, rd, solve_stage, status, st));
    return RLHC_OK;
  };
  int rc;
  if (method == RLHC_CHOLQR2 || method == RLHC_SCHOLQR3) {
    // [W, Y] = (S)CholeskyQR(X): G = X^T X (+ s I), Y = Cholesky, W = X Y^{-1}
    CUDA_TRY(launch_gram(X, ldx, m, ni, a.part, a.G, st));
    if (method == RLHC_SCHOLQR3) CUDA_TRY(launch_shift_diag(a.G, ni, m, st));
    if ((rc = chol(a.Y, a.rdY, RLHC_STAGE_CHOL0))) return rc;
    if ((rc = solve_pass(X, ldx, a.Y, a.rdY, nullptr, nullptr, a.G, true))) return rc;
    if ((rc = chol(a.D, a.Di, RLHC_STAGE_CHOL1))) return rc;
    if (method == RLHC_CHOLQR2) {  // [Q, Z] = CholeskyQR(W), R = Z Y
      if ((rc = solve_pass(Q, ldq, a.D, a.Di, nullptr, nullptr, nullptr))) return rc;
      CUDA_TRY(launch_trmm_uu(a.D, a.Y, ni, R, st));
    } else {  // [Q, Z] = CholeskyQR2(W), R = J (D Y)
      if ((rc = solve_pass(Q, ldq, a.D, a.Di, nullptr, nullptr, a.G))) return rc;
      if ((rc = chol(a.J, a.Ji, RLHC_STAGE_CHOL2))) return rc;
      if ((rc = solve_pass(Q, ldq, a.J, a.Ji, nullptr, nullptr, nullptr))) return rc;
      CUDA_TRY(launch_trmm_uu(a.D, a.Y, ni, a.N, st));
      CUDA_TRY(launch_trmm_uu(a.J, a.N, ni, R, st));
    }
  } else if (method == RLHC_LUC2) {
    // PX = LU, L (into Q), G = L^T L, S = Cholesky(G), Y = S U (diag > 0, R#23), W = X Y^{-1}
    if ((rc = run_tslu(X, m, n, ldx, 0, cfg, a.t, Q, ldq, piv, a.U, a.L11, st))) return rc;
    if (!tslw_cfg(cfg, m, n)) {
      CUDA_TRY(launch_fill_i32(a.pivpos, m, -1, st));
      CUDA_TRY(launch_pivpos(piv, ni, 0, m, a.pivpos, st));
      if ((rc = solve_pass(X, ldx, a.U, a.t.rd, a.pivpos, a.L11, nullptr))) return rc;
    }
    CUDA_TRY(launch_gram(Q, ldq, m, ni, a.part, a.G, st));
    if ((rc = chol(a.S, a.Di, RLHC_STAGE_CHOL0))) return rc;
    CUDA_TRY(launch_trmm_uu(a.S, a.U, ni, a.Y, st));
    CUDA_TRY(launch_flip_neg_rows(a.Y, ni, st));
    CUDA_TRY(launch_rdiag(a.Y, ni, n, a.rdY, RLHC_STAGE_SOLVE_Y, status, st));
    if ((rc = solve_pass(X, ldx, a.Y, a.rdY, nullptr, nullptr, a.G, true))) return rc;
    if ((rc = chol(a.D, a.Di, RLHC_STAGE_CHOL1))) return rc;
    if ((rc = solve_pass(Q, ldq, a.D, a.Di, nullptr, nullptr, nullptr))) return rc;
    CUDA_TRY(launch_trmm_uu(a.D, a.Y, ni, R, st));
  } else {
    // RHC: K = Omega_2 Omega_1 X, [H, Y] = HouseholderQR(K) (diag > 0, R#22), W = X Y^{-1},
    // [Q, Z] = CholeskyQR(W), R = Z Y
    CUDA_TRY(launch_sketch_count(X, ldx, m, ni, 0, (int)s1, seed, a.plan, a.Lt, nullptr, nullptr, st));
    CUDA_TRY(launch_sketch_gauss(a.Lt, n, s1, ni, 0, (int)s2, seed, 1u, a.part, a.Ls, st));
    CUDA_TRY(launch_hqr(a.Ls, (int)s2, ni, n, nullptr, a.Y, a.work, status, st));
    CUDA_TRY(launch_flip_neg_rows(a.Y, ni, st));
    CUDA_TRY(launch_rdiag(a.Y, ni, n, a.rdY, RLHC_STAGE_SOLVE_Y, status, st));
    if ((rc = solve_pass(X, ldx, a.Y, a.rdY, nullptr, nullptr, a.G, true))) return rc;
    if ((rc = chol(a.D, a.Di, RLHC_STAGE_CHOL1))) return rc;
    if ((rc = solve_pass(Q, ldq, a.D, a.Di, nullptr, nullptr, nullptr))) return rc;
    CUDA_TRY(launch_trmm_uu(a.D, a.Y, ni, R, st));
  }
  CUDA_TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

int check_common(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R, int64_t* piv,
                 void* ws, rlhc_info_t* info) {
  if (!X || !Q || !R || !piv || !ws || !info) return fail(RLHC_EINVAL, "null pointer argument");
  if (n < 1 || m < n) return fail(RLHC_EINVAL, "need m >= n >= 1");
  if (m > 0x7fffffffLL) return fail(RLHC_EINVAL, "m must be < 2^31 (int32 row ids)");
  if (ldx < n || ldq < n) return fail(RLHC_EINVAL, "leading dimension < n");
  if (((uintptr_t)ws) & 255) return fail(RLHC_EINVAL, "workspace must be 256-byte aligned");
  if (overlaps(X, (size_t)((m - 1) * ldx + n) * 8, Q, (size_t)((m - 1) * ldq + n) * 8))
    return fail(RLHC_EINVAL, "Q overlaps X");
  return RLHC_OK;
}

}  // namespace

extern "C" {

void rlhc_default_tslu_cfg(int64_t m, int64_t n, rlhc_tslu_cfg* cfg) {
  (void)m;
  if (!cfg) return;
  // the warp tournament (tslw.cu): 16-column panels, 128-row leaves, nodes of 8 children
  cfg->panel = (int)std::min<int64_t>(std::max<int64_t>(n, 1), kTslwPanel);
  cfg->leaf_rows = 128;
  cfg->arity = 8;
}

size_t rlhc_workspace_size(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2, const rlhc_tslu_cfg* cfgp) {
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(m, n, &cfg);
  if (n < 1 || m < n || !cfg_ok(cfg, m, n)) return 0;
  if (algo == RLHC_SLHC3 && (s_or_s1 < n || s_or_s1 > m)) return 0;
  if (algo == RLHC_SSLHC3 && (s2 < n || s_or_s1 < s2 || s_or_s1 > m)) return 0;
  if (algo != RLHC_SLHC3 && algo != RLHC_SSLHC3) return 0;
  Carver c(nullptr);
  AlgoWs a;
  carve_algo(c, algo, m, n, s_or_s1, s2, cfg, a);
  return c.used;
}

size_t rlhc_method_workspace_size(int method, int64_t m, int64_t n, int64_t s1, int64_t s2, const rlhc_tslu_cfg* cfgp) {
  if (method < RLHC_CHOLQR2 || method > RLHC_RHC || n < 1 || m < n) return 0;
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(m, n, &cfg);
  if (!cfg_ok(cfg, m, n)) return 0;
  if (method == RLHC_RHC && (s2 < n || s1 < s2 || s1 > m)) return 0;
  Carver c(nullptr);
  AlgoWs a;
  carve_algo(c, RLHC_SSLHC3, m, n, std::max(s1, n), std::max(s2, n), cfg, a);
  return c.used;
}

static int method_entry(int method, const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2,
                        uint64_t seed, const rlhc_tslu_cfg* cfgp, double* Q, int64_t ldq, double* R, int64_t* piv,
                        void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  int rc = check_common(X, m, n, ldx, Q, ldq, R, piv, ws, info);
  if (rc) return rc;
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(m, n, &cfg);
  if (!cfg_ok(cfg, m, n)) return fail(RLHC_EINVAL, "unsupported tslu configuration (see rlhc_default_tslu_cfg)");
  if (method == RLHC_RHC && (s2 < n || s1 < s2 || s1 > m)) return fail(RLHC_EINVAL, "need n <= s2 <= s1 <= m");
  size_t need = rlhc_method_workspace_size(method, m, n, s1, s2, &cfg);
  if (ws_bytes < need) return fail(RLHC_EWORKSPACE, "workspace too small");
  Carver c(ws);
  AlgoWs a;
  carve_algo(c, RLHC_SSLHC3, m, n, std::max(s1, n), std::max(s2, n), cfg, a);
  return run_method(method, X, m, n, ldx, s1, s2, seed, cfg, Q, ldq, R, piv, a, info, (cudaStream_t)stream);
}

int rlhc_cholqr2(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R, void* ws,
                 size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  int64_t dummy_piv;
  return method_entry(RLHC_CHOLQR2, X, m, n, ldx, n, n, 0, nullptr, Q, ldq, R, &dummy_piv, ws, ws_bytes, info, stream);
}
int rlhc_scholqr3(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R, void* ws,
                  size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  int64_t dummy_piv;
  return method_entry(RLHC_SCHOLQR3, X, m, n, ldx, n, n, 0, nullptr, Q, ldq, R, &dummy_piv, ws, ws_bytes, info,
                      stream);
}
int rlhc_luc2(const double* X, int64_t m, int64_t n, int64_t ldx, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq,
              double* R, int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  return method_entry(RLHC_LUC2, X, m, n, ldx, n, n, 0, cfg, Q, ldq, R, piv, ws, ws_bytes, info, stream);
}
int rlhc_rhc(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed, double* Q,
             int64_t ldq, double* R, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  int64_t dummy_piv;
  return method_entry(RLHC_RHC, X, m, n, ldx, s1, s2, seed, nullptr, Q, ldq, R, &dummy_piv, ws, ws_bytes, info,
                      stream);
}

static int algo_entry(int algo, const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s_or_s1, int64_t s2,
                      uint64_t seed, const rlhc_tslu_cfg* cfgp, double* Q, int64_t ldq, double* R, int64_t* piv,
                      void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  int rc = check_common(X, m, n, ldx, Q, ldq, R, piv, ws, info);
  if (rc) return rc;
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(m, n, &cfg);
  if (!cfg_ok(cfg, m, n)) return fail(RLHC_EINVAL, "unsupported tslu configuration (see rlhc_default_tslu_cfg)");
  if (algo == RLHC_SLHC3 && (s_or_s1 < n || s_or_s1 > m)) return fail(RLHC_EINVAL, "need n <= s <= m");
  if (algo == RLHC_SSLHC3 && (s2 < n || s_or_s1 < s2 || s_or_s1 > m))
    return fail(RLHC_EINVAL, "need n <= s2 <= s1 <= m");
  size_t need = rlhc_workspace_size(algo, m, n, s_or_s1, s2, &cfg);
  if (ws_bytes < need) return fail(RLHC_EWORKSPACE, "workspace too small");
  Carver c(ws);
  AlgoWs a;
  carve_algo(c, algo, m, n, s_or_s1, s2, cfg, a);
  return run_algo(algo, X, m, n, ldx, s_or_s1, s2, seed, cfg, Q, ldq, R, piv, a, info, (cudaStream_t)stream);
}

int rlhc_slhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s, uint64_t seed, const rlhc_tslu_cfg* cfg,
               double* Q, int64_t ldq, double* R, int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info,
               rlhc_stream_t stream) {
  return algo_entry(RLHC_SLHC3, X, m, n, ldx, s, 0, seed, cfg, Q, ldq, R, piv, ws, ws_bytes, info, stream);
}

int rlhc_sslhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed,
                const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq, double* R, int64_t* piv, void* ws, size_t ws_bytes,
                rlhc_info_t* info, rlhc_stream_t stream) {
  return algo_entry(RLHC_SSLHC3, X, m, n, ldx, s1, s2, seed, cfg, Q, ldq, R, piv, ws, ws_bytes, info, stream);
}

// ---- host-buffer pipeline: count independent problems streamed through double-buffered
// device copies (H2D of i+1 and D2H of i-1 on internal copy streams while i computes)
struct HostPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
};
static cudaError_t host_pipe(HostPipe** out) {
  static thread_local std::array<HostPipe, 64> per_dev;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  HostPipe& hp = per_dev[dev];
  if (!hp.h2d) {
    if ((e = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking))) return e;
    if ((e = cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking))) return e;
    for (int b = 0; b < 2; b++) {
      if ((e = cudaEventCreateWithFlags(&hp.ev_h2d[b], cudaEventDisableTiming))) return e;
      if ((e = cudaEventCreateWithFlags(&hp.ev_comp[b], cudaEventDisableTiming))) return e;
      if ((e = cudaEventCreateWithFlags(&hp.ev_d2h[b], cudaEventDisableTiming))) return e;
    }
  }
  *out = &hp;
  return cudaSuccess;
}
struct PipeWs {
  void* algo_ws;
  size_t algo_bytes;
  double *X[2], *Q[2], *R[2];
  int64_t* piv[2];
  rlhc_info_t* info[2];
};
static size_t pipe_carve(void* ws, int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2,
                         const rlhc_tslu_cfg* cfg, PipeWs& p) {
  p.algo_bytes = rlhc_workspace_size(algo, m, n, s_or_s1, s2, cfg);
  if (!p.algo_bytes) return 0;
  Carver c(ws);
  p.algo_ws = c.take<char>(p.algo_bytes);
  for (int b = 0; b < 2; b++) {
    p.X[b] = c.take<double>((size_t)m * n);
    p.Q[b] = c.take<double>((size_t)m * n);
    p.R[b] = c.take<double>((size_t)n * n);
    p.piv[b] = c.take<int64_t>((size_t)n);
    p.info[b] = c.take<rlhc_info_t>(1);
  }
  return c.used;
}

size_t rlhc_host_pipeline_workspace_size(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2,
                                         const rlhc_tslu_cfg* cfg) {
  PipeWs p;
  return pipe_carve(nullptr, algo, m, n, s_or_s1, s2, cfg, p);
}

int rlhc_host_pipeline(int algo, int64_t count, const double* const* X_host, int64_t m, int64_t n, int64_t s_or_s1,
                       int64_t s2, const uint64_t* seeds, const rlhc_tslu_cfg* cfg, double* const* Q_host,
                       double* const* R_host, int64_t* const* piv_host, rlhc_info_t* info_host, void* ws,
                       size_t ws_bytes, rlhc_stream_t stream) {
  if (algo != RLHC_SLHC3 && algo != RLHC_SSLHC3) return fail(RLHC_EINVAL, "unknown algorithm");
  if (count < 0 || (count > 0 && (!X_host || !seeds || !Q_host || !R_host || !info_host || !ws)))
    return fail(RLHC_EINVAL, "null pointer argument");
  PipeWs p;
  const size_t need = pipe_carve(nullptr, algo, m, n, s_or_s1, s2, cfg, p);
  if (!need) return fail(RLHC_EINVAL, "invalid sizes");
  if (ws_bytes < need) return fail(RLHC_EWORKSPACE, "workspace too small");
  pipe_carve(ws, algo, m, n, s_or_s1, s2, cfg, p);
  HostPipe* hp = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(host_pipe(&hp));
  const size_t xb = (size_t)m * n * sizeof(double), rb = (size_t)n * n * sizeof(double);
  // the copy streams start after the work already queued on `stream`
  CUDA_TRY(cudaEventRecord(hp->ev_d2h[0], st));
  CUDA_TRY(cudaStreamWaitEvent(hp->h2d, hp->ev_d2h[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(hp->d2h, hp->ev_d2h[0], 0));
  for (int64_t i = 0; i < count; i++) {
    const int b = (int)(i & 1);
    if (!X_host[i] || !Q_host[i] || !R_host[i]) return fail(RLHC_EINVAL, "null pointer argument");
    if (i >= 2) CUDA_TRY(cudaStreamWaitEvent(hp->h2d, hp->ev_comp[b], 0));  // X[b] consumed by i-2
    CUDA_TRY(cudaMemcpyAsync(p.X[b], X_host[i], xb, cudaMemcpyHostToDevice, hp->h2d));
    CUDA_TRY(cudaEventRecord(hp->ev_h2d[b], hp->h2d));
    CUDA_TRY(cudaStreamWaitEvent(st, hp->ev_h2d[b], 0));
    if (i >= 2) CUDA_TRY(cudaStreamWaitEvent(st, hp->ev_d2h[b], 0));  // Q[b], R[b] drained for i-2
    int rc = algo_entry(algo, p.X[b], m, n, n, s_or_s1, s2, seeds[i], cfg, p.Q[b], n, p.R[b], p.piv[b], p.algo_ws,
                        p.algo_bytes, p.info[b], stream);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(hp->ev_comp[b], st));
    CUDA_TRY(cudaStreamWaitEvent(hp->d2h, hp->ev_comp[b], 0));
    CUDA_TRY(cudaMemcpyAsync(Q_host[i], p.Q[b], xb, cudaMemcpyDeviceToHost, hp->d2h));
    CUDA_TRY(cudaMemcpyAsync(R_host[i], p.R[b], rb, cudaMemcpyDeviceToHost, hp->d2h));
    if (piv_host && piv_host[i])
      CUDA_TRY(cudaMemcpyAsync(piv_host[i], p.piv[b], (size_t)n * sizeof(int64_t), cudaMemcpyDeviceToHost, hp->d2h));
    CUDA_TRY(cudaMemcpyAsync(info_host + i, p.info[b], sizeof(rlhc_info_t), cudaMemcpyDeviceToHost, hp->d2h));
    CUDA_TRY(cudaEventRecord(hp->ev_d2h[b], hp->d2h));
  }
  // `stream` completes after the last device-to-host copy
  for (int64_t i = std::max<int64_t>(0, count - 2); i < count; i++)
    CUDA_TRY(cudaStreamWaitEvent(st, hp->ev_d2h[i & 1], 0));
  if (count == 0) CUDA_TRY(cudaStreamWaitEvent(st, hp->ev_d2h[0], 0));
  return RLHC_OK;
}

// ---------------------------------------------------------------- per-stage
static size_t getrf_carve(Carver& c, int64_t rows, int64_t n, const rlhc_tslu_cfg& cfg, TsluWs& t, double** tw,
                          int** pivpos) {
  t.status = c.take<unsigned long long>(4);
  carve_tslu(c, rows, n, cfg, t);
  *tw = (cfg.panel < n || tslw_cfg(cfg, rows, n)) ? c.take<double>((size_t)rows * n) : nullptr;
  *pivpos = c.take<int>((size_t)rows);
  return c.used;
}

size_t rlhc_getrf_ts_workspace_size(int64_t rows, int64_t n, const rlhc_tslu_cfg* cfgp) {
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(rows, n, &cfg);
  if (n < 1 || rows < n || !cfg_ok(cfg, rows, n)) return 0;
  Carver c(nullptr);
  TsluWs t;
  double* tw;
  int* pp;
  return getrf_carve(c, rows, n, cfg, t, &tw, &pp);
}

int rlhc_getrf_ts(const double* X, int64_t rows, int64_t n, int64_t ldx, int64_t row0, const rlhc_tslu_cfg* cfgp,
                  int64_t* piv, double* U, double* L11, double* L, int64_t ldl, void* ws, size_t ws_bytes,
                  rlhc_info_t* info, rlhc_stream_t stream) {
  if (!X || !piv || !U || !L11 || !ws || !info) return fail(RLHC_EINVAL, "null pointer argument");
  if (n < 1 || rows < n || ldx < n || (L && ldl < n)) return fail(RLHC_EINVAL, "bad sizes");
  if (row0 != 0) return fail(RLHC_EINVAL, "row0 must be 0 for the single-device entry point");
  if (rows > 0x7fffffffLL) return fail(RLHC_EINVAL, "rows must be < 2^31");
  rlhc_tslu_cfg cfg;
  if (cfgp) cfg = *cfgp; else rlhc_default_tslu_cfg(rows, n, &cfg);
  if (!cfg_ok(cfg, rows, n)) return fail(RLHC_EINVAL, "unsupported tslu configuration");
  size_t need = rlhc_getrf_ts_workspace_size(rows, n, &cfg);
  if (ws_bytes < need) return fail(RLHC_EWORKSPACE, "workspace too small");
  Carver c(ws);
  TsluWs t;
  double* tw;
  int* pivpos;
  getrf_carve(c, rows, n, cfg, t, &tw, &pivpos);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(launch_status_init(t.status, st));
  if (tslw_cfg(cfg, rows, n)) {  // input check folded into the leaves; L straight into the caller's buffer
    int rc = run_tslu(X, rows, n, ldx, row0, cfg, t, L ? L : tw, L ? ldl : n, piv, U, L11, st, true);
    if (rc) return rc;
    CUDA_TRY(launch_status_finish(t.status, info, st));
    return RLHC_OK;
  }
  CUDA_TRY(launch_check_finite(X, rows, (int)n, ldx, t.status, st));
  int rc = run_tslu(X, rows, n, ldx, row0, cfg, t, tw, n, piv, U, L11, st);
  if (rc) return rc;
  if (L) {
    (void)pivpos;
    CUDA_TRY(launch_trsm_blocked(X, ldx, rows, (int)n, (int)n, U, n, t.rd, L, ldl, st));
    CUDA_TRY(launch_pivot_rows(piv, (int)n, row0, rows, L11, L, ldl, st));
  }
  CUDA_TRY(launch_status_finish(t.status, info, st));
  return RLHC_OK;
}

size_t rlhc_sketch_gauss_workspace_size(int64_t rows, int64_t n, int64_t s) {
  if (rows < 1 || n < 1 || s < 1) return 0;
  return al(gauss_partials_bytes(rows, (int)n, (int)s));
}

int rlhc_sketch_gauss(const double* A, int64_t rows, int64_t n, int64_t lda, int64_t row0, int64_t s, uint64_t seed,
                      uint32_t stream_id, double* out, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  if (!A || !out || !ws) return fail(RLHC_EINVAL, "null pointer argument");
  if (rows < 1 || n < 1 || s < 1 || lda < n || row0 < 0) return fail(RLHC_EINVAL, "bad sizes");
  if (ws_bytes < rlhc_sketch_gauss_workspace_size(rows, n, s)) return fail(RLHC_EWORKSPACE, "workspace too small");
  CUDA_TRY(launch_sketch_gauss(A, lda, rows, (int)n, row0, (int)s, seed, stream_id, (double*)ws, out,
                               (cudaStream_t)stream));
  return RLHC_OK;
}

size_t rlhc_sketch_count_workspace_size(int64_t rows, int64_t n, int64_t s1) {
  if (rows < 1 || n < 1 || s1 < 1) return 0;
  return al(cs_plan_bytes(rows, (int)s1));
}

int rlhc_sketch_count(const double* A, int64_t rows, int64_t n, int64_t lda, int64_t row0, int64_t s1, uint64_t seed,
                      double* out, int32_t* bucket, int8_t* sign, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  if (!A || !out || !ws) return fail(RLHC_EINVAL, "null pointer argument");
  if (rows < 1 || n < 1 || s1 < 1 || lda < n || row0 < 0 || rows > 0x7fffffffLL || s1 > 65536)
    return fail(RLHC_EINVAL, "bad sizes");
  if (ws_bytes < rlhc_sketch_count_workspace_size(rows, n, s1)) return fail(RLHC_EWORKSPACE, "workspace too small");
  CUDA_TRY(launch_sketch_count(A, lda, rows, (int)n, row0, (int)s1, seed, ws, out, bucket, sign, (cudaStream_t)stream));
  return RLHC_OK;
}

size_t rlhc_gram_workspace_size(int64_t rows, int64_t n) {
  if (rows < 1 || n < 1) return 0;
  return al(gram_partials_bytes(rows, (int)n));
}

int rlhc_gram(const double* A, int64_t rows, int64_t n, int64_t lda, double* G, void* ws, size_t ws_bytes,
              rlhc_stream_t stream) {
  if (!A || !G || !ws) return fail(RLHC_EINVAL, "null pointer argument");
  if (rows < 1 || n < 1 || lda < n) return fail(RLHC_EINVAL, "bad sizes");
  if (ws_bytes < rlhc_gram_workspace_size(rows, n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  CUDA_TRY(launch_gram(A, lda, rows, (int)n, (double*)ws, G, (cudaStream_t)stream));
  return RLHC_OK;
}

size_t rlhc_trsm_apply_workspace_size(int64_t rows, int64_t n) {
  if (rows < 1 || n < 1) return 0;
  return al(256) + al((size_t)n * 8) + al((size_t)n * n * 8) + al(gram_partials_bytes(rows, (int)n)) +
         al(ts_gemm_pack_bytes((int)n, (int)n));
}

int rlhc_trsm_apply(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int mode, double* out,
                    int64_t ldo, double* G_out, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  if (!A || !T || !out || !ws || !info) return fail(RLHC_EINVAL, "null pointer argument");
  if (rows < 1 || n < 1 || lda < n || ldo < n) return fail(RLHC_EINVAL, "bad sizes");
  if (mode != RLHC_SUBST && mode != RLHC_INV_GEMM) return fail(RLHC_EINVAL, "bad mode");
  if (out != A && overlaps(A, (size_t)((rows - 1) * lda + n) * 8, out, (size_t)((rows - 1) * ldo + n) * 8))
    return fail(RLHC_EINVAL, "out partially overlaps A");
  if (out == A && lda != ldo) return fail(RLHC_EINVAL, "in place needs lda == ldo");
  if (ws_bytes < rlhc_trsm_apply_workspace_size(rows, n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  Carver c(ws);
  unsigned long long* status = c.take<unsigned long long>(4);
  double* rd = c.take<double>((size_t)n);
  double* Ti = c.take<double>((size_t)n * n);
  double* part = c.take<double>(gram_partials_bytes(rows, (int)n) / 8 + 1);
  double* bpack = c.take<double>(ts_gemm_pack_bytes((int)n, (int)n) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(launch_status_init(status, st));
  CUDA_TRY(launch_rdiag(T, (int)n, n, rd, RLHC_STAGE_SOLVE_Y, status, st));
  if (mode == RLHC_SUBST && subst_ms_ok((int)n)) {
    CUDA_TRY(launch_subst_ms(A, lda, rows, (int)n, T, n, out, ldo, nullptr, nullptr, st));
  } else if (mode == RLHC_SUBST && subst_wide_ok((int)n)) {
    CUDA_TRY(launch_subst_wide(A, lda, rows, (int)n, T, n, out, ldo, st));
  } else if (mode == RLHC_SUBST) {
    CUDA_TRY(launch_trsm_rows(A, lda, rows, (int)n, (int)n, T, n, rd, out, ldo, nullptr, nullptr, 0, st));
  } else {
    CUDA_TRY(launch_tri_inv(T, (int)n, Ti, st));
    CUDA_TRY(launch_ts_gemm(nullptr, 0, out, ldo, A, lda, Ti, n, rows, (int)n, (int)n, true, false, bpack, st));
  }
  if (G_out) CUDA_TRY(launch_gram(out, ldo, rows, (int)n, part, G_out, st));
  CUDA_TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}

size_t rlhc_hqr_workspace_size(int64_t s, int64_t n) {
  if (s < n || n < 1) return 0;
  return al(256) + al(hqr_ws_bytes((int)s, (int)n));
}

int rlhc_hqr_r(const double* A, int64_t s, int64_t n, int64_t lda, const double* sgn_ref, double* S, void* ws,
               size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream) {
  if (!A || !S || !ws || !info) return fail(RLHC_EINVAL, "null pointer argument");
  if (n < 1 || s < n || lda < n) return fail(RLHC_EINVAL, "bad sizes");
  if (ws_bytes < rlhc_hqr_workspace_size(s, n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  Carver c(ws);
  unsigned long long* status = c.take<unsigned long long>(4);
  double* work = c.take<double>(hqr_ws_bytes((int)s, (int)n) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(launch_status_init(status, st));
  CUDA_TRY(launch_hqr(A, (int)s, (int)n, lda, sgn_ref, S, work, status, st));
  CUDA_TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}

int rlhc_cholesky(const double* G, int64_t n, double* Rout, int stage, rlhc_info_t* info, rlhc_stream_t stream) {
  if (!G || !Rout || !info) return fail(RLHC_EINVAL, "null pointer argument");
  if (n < 1 || n > 4096) return fail(RLHC_EINVAL, "bad size");
  // status and working copy live in the caller's info / output buffers: the status
  // word is kept in info->index's storage until the final decode
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = (unsigned long long*)&info->index;
  if (chol_ws_bytes((int)n) > 200 * 1024) return fail(RLHC_EINVAL, "rlhc_cholesky entry point supports n <= 110");
  CUDA_TRY(launch_status_init(status, st));
  CUDA_TRY(launch_chol(G, (int)n, Rout, nullptr, stage, status, st));
  CUDA_TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}

const char* rlhc_version(void) { return "rlhc-b200 0.1 (sm_100a, fp64 DMMA)"; }

uint64_t rlhc_launch_count(void) { return (uint64_t)launch_count(); }

void rlhc_stage_timing(int enable) {
  std::lock_guard<std::mutex> g(g_prof.mu);
  g_prof.enabled = enable != 0;
  if (!g_prof.enabled) {
    for (auto& ms : g_prof.pending) g_prof.pool.push_back(ms);
    g_prof.pending.clear();
  }
}

int rlhc_stage_times(double* ms, int max_stages) {
  std::lock_guard<std::mutex> g(g_prof.mu);
  int calls = 0;
  for (auto& ev : g_prof.pending) {
    if (cudaEventSynchronize(ev[kStages]) != cudaSuccess) return -1;
    for (int k = 0; k < kStages && k < max_stages; k++) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev[k], ev[k + 1]) != cudaSuccess) return -1;
      ms[k] += t;
    }
    g_prof.pool.push_back(ev);
    calls++;
  }
  g_prof.pending.clear();
  return calls;
}

const char* rlhc_stage_name(int k) { return (k >= 0 && k < kStages) ? kStageNames[k] : ""; }
const char* rlhc_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

// ---------------------------------------------------------------- CUDA graphs
struct rlhc_graph_s {
  cudaGraphExec_t exec;
};

extern "C" {

int rlhc_graph_begin(rlhc_stream_t stream) {
  if (!stream) return fail(RLHC_EINVAL, "graph capture needs a non-default stream");
  CUDA_TRY(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return RLHC_OK;
}

int rlhc_graph_end(rlhc_stream_t stream, rlhc_graph_t* graph) {
  if (!stream || !graph) return fail(RLHC_EINVAL, "null argument");
  *graph = nullptr;
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamEndCapture((cudaStream_t)stream, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    g_last_error = std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e);
    return RLHC_ECUDA;
  }
  *graph = new rlhc_graph_s{ex};
  return RLHC_OK;
}

int rlhc_graph_launch(rlhc_graph_t graph, rlhc_stream_t stream) {
  if (!graph) return fail(RLHC_EINVAL, "null graph");
  CUDA_TRY(cudaGraphLaunch(graph->exec, (cudaStream_t)stream));
  return RLHC_OK;
}

void rlhc_graph_destroy(rlhc_graph_t graph) {
  if (!graph) return;
  cudaGraphExecDestroy(graph->exec);
  delete graph;
}

}  // extern "C"
