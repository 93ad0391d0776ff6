// dist_blocks.cu -- C ABI building blocks of the row-sharded (multi-GPU) SLHC3 / SSLHC3
// (DESIGN.md section 7).  The orchestration (which rows each rank owns, the
// all-gather of tournament candidates, the all-reduces of sketches and Grams) lives in
// paper_2412_06551_b200/dist.py on top of torch.distributed; every arithmetic step is
// one of the calls below or an existing stage entry point.
#include <string>

#include "common.cuh"
#include "kernels.cuh"

using namespace rlhc;

namespace rlhc {

// out[t][c] = src[(ids[t] - row0)][c0 + c] for the pivots this rank owns, 0 otherwise
// (so an all-reduce SUM of `out` over ranks yields the pivot rows exactly).
__global__ void owned_rows_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t row0,
                                  const int* __restrict__ ids, int w, int c0, int ncols, double* __restrict__ out) {
  const int t = blockIdx.x;
  if (t >= w) return;
  const int64_t lr = (int64_t)ids[t] - row0;
  const bool own = ids[t] >= 0 && lr >= 0 && lr < rows;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) out[(int64_t)t * ncols + c] = own ? src[lr * lds + c0 + c] : 0.0;
}
__global__ void owned_rows64_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t row0,
                                    const int64_t* __restrict__ ids, int w, int c0, int ncols, double* __restrict__ out) {
  const int t = blockIdx.x;
  if (t >= w) return;
  const int64_t lr = ids[t] - row0;
  const bool own = lr >= 0 && lr < rows;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) out[(int64_t)t * ncols + c] = own ? src[lr * lds + c0 + c] : 0.0;
}
__global__ void set_int_kernel(int* p, int v) { *p = v; }

}  // namespace rlhc

namespace {
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
int kw(int panel) { return panel <= 16 ? 16 : (panel <= 32 ? 32 : 64); }
int fail(int code, const char* msg) { set_last_error(msg); return code; }
#define TRY(x)                                                        \
  do {                                                                \
    cudaError_t e_ = (x);                                             \
    if (e_ != cudaSuccess) {                                          \
      set_last_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
      return RLHC_ECUDA;                                              \
    }                                                                 \
  } while (0)

struct LevelBufs {
  int* ids[2];
  int* cnt[2];
  double* vals[2];
};
size_t level_bytes(int64_t slots, int W) {
  return 2 * (al(slots * W * 4) + al((2 * slots + 64) * 4) + al(slots * W * W * 8));
}
LevelBufs carve_levels(void* ws, int64_t slots, int W) {
  LevelBufs b;
  char* p = (char*)ws;
  for (int k = 0; k < 2; k++) {
    b.ids[k] = (int*)p; p += al(slots * W * 4);
    b.cnt[k] = (int*)p; p += al((2 * slots + 64) * 4);  // warp tree: counts + arrival counters
    b.vals[k] = (double*)p; p += al(slots * W * W * 8);
  }
  return b;
}
// reduce `nslots` slots in buffer `cur` down to `target` (node levels; nslots / target a
// power of the arity, or target = 1), returns the final buffer index.  rsrc (local rows): the
// levels read candidate rows from it and only the final level carries values; else every
// slot carries values (slots gathered from other ranks)
int reduce_levels(LevelBufs& b, int cur, int nslots, int arity, int w, int W, cudaStream_t st, int* out_cur,
                  const RowSrc* rsrc = nullptr, int target = 1) {
  while (nslots > target) {
    const int nout = (nslots + arity - 1) / arity;
    TRY(launch_tslu_node(W, b.ids[cur], b.cnt[cur], rsrc ? nullptr : b.vals[cur], nslots, arity, w, b.ids[cur ^ 1],
                         b.cnt[cur ^ 1], (rsrc && nout > target) ? nullptr : b.vals[cur ^ 1], st, nullptr, rsrc));
    nslots = nout;
    cur ^= 1;
  }
  *out_cur = cur;
  return RLHC_OK;
}
int copy_slot(LevelBufs& b, int cur, int W, int* out_ids, int* out_cnt, double* out_vals, cudaStream_t st,
              int64_t k = 1) {
  TRY(cudaMemcpyAsync(out_ids, b.ids[cur], k * W * 4, cudaMemcpyDeviceToDevice, st));
  TRY(cudaMemcpyAsync(out_cnt, b.cnt[cur], k * 4, cudaMemcpyDeviceToDevice, st));
  TRY(cudaMemcpyAsync(out_vals, b.vals[cur], (size_t)k * W * W * 8, cudaMemcpyDeviceToDevice, st));
  return RLHC_OK;
}
// levels from `leaves` slots down to `k` (-1: leaves / k is not a power of the arity)
int levels_to(int64_t leaves, int64_t k, int arity) {
  if (k < 1 || leaves % k) return -1;
  int64_t q = leaves / k;
  int lev = 0;
  while (q > 1) {
    if (q % arity) return -1;
    q /= arity;
    lev++;
  }
  return lev;
}
bool cfg_valid(const rlhc_tslu_cfg* c, int64_t w) {
  return c && c->panel >= 1 && c->panel <= 64 && w >= 1 && w <= c->panel && c->arity >= 2 &&
         c->leaf_rows >= 1 && c->leaf_rows <= select_rows(kw(c->panel)) &&
         (int64_t)c->arity * c->panel <= select_rows(kw(c->panel));
}
}  // namespace

extern "C" {

size_t rlhc_tslu_local_workspace_size(int64_t rows, int64_t nslots_in, const rlhc_tslu_cfg* cfg) {
  if (!cfg || rows < 0 || nslots_in < 0) return 0;
  const int W = kw(cfg->panel);
  const int64_t slots = std::max<int64_t>(std::max<int64_t>(1, ceil_div<int64_t>(rows, cfg->leaf_rows)), nslots_in);
  return level_bytes(slots, W);
}

int64_t rlhc_tslu_local_slots(int64_t rows_local, const rlhc_tslu_cfg* cfg) {
  if (!cfg || cfg->leaf_rows < 1 || cfg->arity < 2 || rows_local < 1) return 0;
  int64_t k = ceil_div<int64_t>(rows_local, cfg->leaf_rows);
  while (k % cfg->arity == 0) k /= cfg->arity;
  return k;
}

int rlhc_tslu_reduce_to(const double* src, int64_t lds, int64_t rows, int64_t row0, int64_t p0, int64_t w,
                        const uint8_t* chosen, const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids,
                        int* out_cnt, double* out_vals, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  if (!src || !out_ids || !out_cnt || !out_vals || !ws || rows < 1) return fail(RLHC_EINVAL, "bad arguments");
  if (!cfg_valid(cfg, w)) return fail(RLHC_EINVAL, "bad tslu configuration");
  if (ws_bytes < rlhc_tslu_local_workspace_size(rows, 0, cfg)) return fail(RLHC_EWORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int W = kw(cfg->panel);
  const int nleaves = (int)ceil_div<int64_t>(rows, cfg->leaf_rows);
  const int lev = nslots_out == 1 ? -1 : levels_to(nleaves, nslots_out, cfg->arity);
  if (nslots_out != 1 && lev < 0)
    return fail(RLHC_EINVAL, "the rank's leaves do not split into nslots_out complete subtrees");
  LevelBufs b = carve_levels(ws, nleaves, W);
  if (cfg->leaf_rows == 128 && cfg->arity >= 2 && cfg->arity <= 8 && w <= 16) {
    // the warp tournament (the default contract): every local level in one launch
    TRY(run_tslw_local_tree(src, lds, rows, row0, (int)p0, (int)w, chosen, cfg->arity, lev, b.ids, b.cnt, b.vals,
                            out_ids, out_cnt, out_vals, st));
    return RLHC_OK;
  }
  const int target = (int)nslots_out;
  TRY(launch_tslu_leaf(W, cfg->leaf_rows, src, lds, rows, row0, (int)p0, (int)w, chosen, b.ids[0], b.cnt[0],
                       nleaves == target ? b.vals[0] : nullptr, st));
  const RowSrc rsrc{src, lds, row0, (int)p0};
  int cur = 0;
  int rc = reduce_levels(b, 0, nleaves, cfg->arity, (int)w, W, st, &cur, &rsrc, target);
  if (rc) return rc;
  return copy_slot(b, cur, W, out_ids, out_cnt, out_vals, st, target);
}

int rlhc_tslw_schur_reduce_to(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl,
                              int64_t row0, int64_t p0, const double* U, const uint8_t* chosen,
                              const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids, int* out_cnt,
                              double* out_vals, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  bool checked = false;
  return tslw_schur_reduce_to_impl(X, rows, n, ldx, L, ldl, row0, p0, U, chosen, cfg, nslots_out, out_ids, out_cnt,
                                   out_vals, nullptr, &checked, ws, ws_bytes, (cudaStream_t)stream);
}

int rlhc_tslu_reduce(const double* src, int64_t lds, int64_t rows, int64_t row0, int64_t p0, int64_t w,
                     const uint8_t* chosen, const rlhc_tslu_cfg* cfg, int* out_ids, int* out_cnt, double* out_vals,
                     void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  return rlhc_tslu_reduce_to(src, lds, rows, row0, p0, w, chosen, cfg, 1, out_ids, out_cnt, out_vals, ws, ws_bytes,
                             stream);
}

int rlhc_tslu_combine(const int* in_ids, const int* in_cnt, const double* in_vals, int64_t nslots, int64_t w,
                      const rlhc_tslu_cfg* cfg, int* out_ids, int* out_cnt, double* out_vals, void* ws, size_t ws_bytes,
                      rlhc_stream_t stream) {
  if (!in_ids || !in_cnt || !in_vals || !out_ids || !out_cnt || !out_vals || !ws || nslots < 1)
    return fail(RLHC_EINVAL, "bad arguments");
  if (!cfg_valid(cfg, w)) return fail(RLHC_EINVAL, "bad tslu configuration");
  if (ws_bytes < rlhc_tslu_local_workspace_size(0, nslots, cfg)) return fail(RLHC_EWORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int W = kw(cfg->panel);
  LevelBufs b = carve_levels(ws, nslots, W);
  TRY(cudaMemcpyAsync(b.ids[0], in_ids, nslots * W * 4, cudaMemcpyDeviceToDevice, st));
  TRY(cudaMemcpyAsync(b.cnt[0], in_cnt, nslots * 4, cudaMemcpyDeviceToDevice, st));
  TRY(cudaMemcpyAsync(b.vals[0], in_vals, (size_t)nslots * W * W * 8, cudaMemcpyDeviceToDevice, st));
  int cur = 0;
  int rc = reduce_levels(b, 0, (int)nslots, cfg->arity, (int)w, W, st, &cur);
  if (rc) return rc;
  return copy_slot(b, cur, W, out_ids, out_cnt, out_vals, st);
}

int rlhc_owned_rows(const double* src, int64_t lds, int64_t rows, int64_t row0, const int* ids32, const int64_t* ids64,
                    int64_t w, int64_t c0, int64_t ncols, double* out, rlhc_stream_t stream) {
  if (!src || !out || (!ids32 && !ids64) || w < 1 || ncols < 1) return fail(RLHC_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  note_launch();
  if (ids32)
    owned_rows_kernel<<<(int)w, 128, 0, st>>>(src, lds, rows, row0, ids32, (int)w, (int)c0, (int)ncols, out);
  else
    owned_rows64_kernel<<<(int)w, 128, 0, st>>>(src, lds, rows, row0, ids64, (int)w, (int)c0, (int)ncols, out);
  TRY(cudaGetLastError());
  return RLHC_OK;
}

size_t rlhc_tslu_panel_workspace_size(int64_t n) { return al(256) + al(64) + al((size_t)n * 8); }

int rlhc_tslu_panel_factor_rows(const double* prow, const int* ids, int64_t p0, int64_t w, int64_t n, int64_t row0,
                                int64_t rows, double* U, int64_t* piv, uint8_t* chosen, void* ws, size_t ws_bytes,
                                rlhc_info_t* info, rlhc_stream_t stream) {
  if (!prow || !ids || !U || !piv || !ws || !info || w < 1 || w > 64 || p0 < 0 || p0 + w > n)
    return fail(RLHC_EINVAL, "bad arguments");
  if (ws_bytes < rlhc_tslu_panel_workspace_size(n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* p = (char*)ws;
  unsigned long long* status = (unsigned long long*)p; p += al(256);
  int* cntw = (int*)p; p += al(64);
  double* rd = (double*)p;
  TRY(launch_status_init(status, st));
  note_launch();
  set_int_kernel<<<1, 1, 0, st>>>(cntw, (int)w);
  TRY(launch_tslu_panel_factor(prow - p0, n - p0, rows, row0, (int)p0, (int)w, (int)n, ids, cntw, U, piv, chosen,
                               nullptr, status, st, 1));
  TRY(launch_rdiag(U + p0 * n + p0, (int)w, n, rd + p0, RLHC_STAGE_LU, status, st));
  TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}

size_t rlhc_tslu_eliminate_workspace_size(int64_t n) { return al(256) + al((size_t)n * 8); }

int rlhc_tslu_eliminate(const double* src, int64_t lds, int64_t rows, int64_t p0, int64_t w, int64_t n,
                        const double* U, double* dst, int64_t ldd, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  if (!src || !dst || !U || !ws || w < 1 || p0 + w > n) return fail(RLHC_EINVAL, "bad arguments");
  if (ws_bytes < rlhc_tslu_eliminate_workspace_size(n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  if (rows < 1 || p0 + w == n) return RLHC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = (unsigned long long*)ws;
  double* rd = (double*)((char*)ws + al(256));
  TRY(launch_status_init(status, st));
  TRY(launch_rdiag(U + p0 * n + p0, (int)w, n, rd, RLHC_STAGE_LU, status, st));
  TRY(launch_trsm_rows(src + p0, lds, rows, (int)(n - p0), (int)w, U + p0 * n + p0, n, rd, dst + p0, ldd, nullptr,
                       nullptr, 0, st));
  return RLHC_OK;
}

int rlhc_tslw_schur(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl, int64_t p0,
                    const double* U, rlhc_stream_t stream) {
  if (!X || !L || !U || rows < 1 || n < 1 || ldx < n || ldl < n || p0 < 0 || p0 >= n || p0 % 16)
    return fail(RLHC_EINVAL, "bad arguments");
  TRY(launch_tslw_schur(X, ldx, L, ldl, rows, (int)p0, (int)std::min<int64_t>(16, n - p0), (int)n, U,
                        (cudaStream_t)stream));
  return RLHC_OK;
}

int rlhc_tslw_owned_rows(const double* X, int64_t ldx, const double* L, int64_t ldl, int64_t rows, int64_t row0,
                         const int* ids, int64_t cnt, int64_t p0, int64_t n, const double* U, double* T,
                         rlhc_stream_t stream) {
  if (!X || !L || !ids || !U || !T || rows < 0 || n < 1 || cnt < 0 || cnt > 16 || p0 < 0 || p0 >= n)
    return fail(RLHC_EINVAL, "bad arguments");
  if (cnt == 0) return RLHC_OK;
  TRY(launch_tslw_owned(X, ldx, L, ldl, rows, row0, ids, (int)cnt, (int)p0, (int)n, U, T, (cudaStream_t)stream));
  return RLHC_OK;
}

int rlhc_tslw_finish(double* L, int64_t ldl, int64_t rows, int64_t row0, int64_t n, const double* U,
                     const int64_t* piv, rlhc_stream_t stream) {
  if (!L || !U || !piv || rows < 1 || n < 1 || ldl < n) return fail(RLHC_EINVAL, "bad arguments");
  TRY(launch_tslw_finish(L, ldl, rows, row0, (int)n, U, piv, (cudaStream_t)stream));
  return RLHC_OK;
}

size_t rlhc_lfactor_workspace_size(int64_t rows, int64_t n) {
  return al(256) + al((size_t)n * 8) + al(rowsolve_partials_bytes(std::max<int64_t>(rows, n), (int)n));
}

// L11 from the pivot rows of X (n x n, pivot order): substitution through U, unit diagonal
int rlhc_l11(const double* Xp, int64_t n, const double* U, double* L11, void* ws, size_t ws_bytes,
             rlhc_stream_t stream) {
  if (!Xp || !U || !L11 || !ws || n < 1) return fail(RLHC_EINVAL, "bad arguments");
  if (ws_bytes < rlhc_lfactor_workspace_size(n, n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = (unsigned long long*)ws;
  double* rd = (double*)((char*)ws + al(256));
  TRY(launch_status_init(status, st));
  TRY(launch_rdiag(U, (int)n, n, rd, RLHC_STAGE_LU, status, st));
  TRY(launch_trsm_rows(Xp, n, n, (int)n, (int)n, U, n, rd, L11, n, nullptr, nullptr, 0, st));
  TRY(launch_l11_fixup(L11, (int)n, st));
  return RLHC_OK;
}

// L rows of this rank's X rows (global ids row0..): substitution through U, pivot rows take L11 rows
int rlhc_lfactor(const double* X, int64_t rows, int64_t n, int64_t ldx, int64_t row0, const double* U, const double* L11,
                 const int64_t* piv, double* L, int64_t ldl, void* ws, size_t ws_bytes, rlhc_stream_t stream) {
  if (!X || !U || !L11 || !piv || !L || !ws || n < 1 || rows < 0) return fail(RLHC_EINVAL, "bad arguments");
  if (ws_bytes < rlhc_lfactor_workspace_size(rows, n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  if (rows == 0) return RLHC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = (unsigned long long*)ws;
  double* rd = (double*)((char*)ws + al(256));
  double* part = (double*)((char*)ws + al(256) + al((size_t)n * 8));
  TRY(launch_status_init(status, st));
  TRY(launch_rdiag(U, (int)n, n, rd, RLHC_STAGE_LU, status, st));
  if (rowsolve_ok((int)n)) {
    TRY(launch_rowsolve(X, ldx, rows, (int)n, U, rd, L, ldl, nullptr, L11, part, nullptr, st));
  } else {
    TRY(launch_trsm_rows(X, ldx, rows, (int)n, (int)n, U, n, rd, L, ldl, nullptr, nullptr, 0, st));
  }
  TRY(launch_pivot_rows(piv, (int)n, row0, rows, L11, L, ldl, st));
  return RLHC_OK;
}

int rlhc_trmm_upper(const double* A, const double* B, int64_t n, double* C, rlhc_stream_t stream) {
  if (!A || !B || !C || n < 1) return fail(RLHC_EINVAL, "bad arguments");
  TRY(launch_trmm_uu(A, B, (int)n, C, (cudaStream_t)stream));
  return RLHC_OK;
}

size_t rlhc_cholesky_workspace_size(int64_t n) { return al(256) + al(chol_ws_bytes((int)n)); }

int rlhc_cholesky_ws(const double* G, int64_t n, double* Rout, int stage, void* ws, size_t ws_bytes, rlhc_info_t* info,
                     rlhc_stream_t stream) {
  if (!G || !Rout || !ws || !info || n < 1) return fail(RLHC_EINVAL, "bad arguments");
  if (ws_bytes < rlhc_cholesky_workspace_size(n)) return fail(RLHC_EWORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = (unsigned long long*)ws;
  double* work = (double*)((char*)ws + al(256));
  TRY(launch_status_init(status, st));
  TRY(launch_chol(G, (int)n, Rout, work, stage, status, st));
  TRY(launch_status_finish(status, info, st));
  return RLHC_OK;
}


}  // extern "C"

namespace rlhc {
int tslw_schur_reduce_to_impl(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl,
                              int64_t row0, int64_t p0, const double* U, const uint8_t* chosen,
                              const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids, int* out_cnt,
                              double* out_vals, unsigned long long* status, bool* checked, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  *checked = false;
  if (!X || !L || !U || !out_ids || !out_cnt || !out_vals || !ws || rows < 1 || n < 1 || ldx < n || ldl < n ||
      p0 < 0 || p0 >= n || p0 % 16)
    return fail(RLHC_EINVAL, "bad arguments");
  const int64_t w = std::min<int64_t>(16, n - p0);
  if (!cfg_valid(cfg, w) || cfg->leaf_rows != 128 || cfg->panel != 16 || cfg->arity < 2 || cfg->arity > 8)
    return fail(RLHC_EINVAL, "bad tslu configuration (the warp contract: 128-row leaves, 16-column panels)");
  if (ws_bytes < rlhc_tslu_local_workspace_size(rows, 0, cfg)) return fail(RLHC_EWORKSPACE, "workspace too small");
  const int nleaves = (int)ceil_div<int64_t>(rows, cfg->leaf_rows);
  const int lev = nslots_out == 1 ? -1 : levels_to(nleaves, nslots_out, cfg->arity);
  if (nslots_out != 1 && lev < 0)
    return fail(RLHC_EINVAL, "the rank's leaves do not split into nslots_out complete subtrees");
  LevelBufs b = carve_levels(ws, nleaves, kw(cfg->panel));
  bool fused = false;
  TRY(run_tslw_schur_local_tree(X, ldx, L, ldl, rows, row0, (int)p0, (int)w, (int)n, U, chosen, cfg->arity, lev,
                                b.ids, b.cnt, b.vals, out_ids, out_cnt, out_vals, status, st, &fused));
  if (fused) {
    *checked = status != nullptr;
    return RLHC_OK;
  }
  int rc = rlhc_tslw_schur(X, rows, n, ldx, L, ldl, p0, U, st);
  if (rc) return rc;
  return rlhc_tslu_reduce_to(L, ldl, rows, row0, p0, w, chosen, cfg, nslots_out, out_ids, out_cnt, out_vals, ws,
                             ws_bytes, st);
}
}  // namespace rlhc
