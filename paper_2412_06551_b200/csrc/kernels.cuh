// kernels.cuh -- launch wrappers of the rLHC sm_100a kernels (internal; not the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/rlhc.h"

namespace rlhc {

int select_rows(int W);
void set_last_error(const std::string& msg);
unsigned long long launch_count();

// tslu.cu
// Root-node outputs of a single-panel factorization (the root's GEPP computes them on the
// way, select.cuh): U written during the select; piv, L11 and 1/diag(U) after it.
struct RootOut {
  double* U;       // n x n, ld n (strict lower part pre-zeroed by the caller)
  int64_t* piv;    // [n] global row ids in pivot order
  double* L11;     // n x n, ld n: multipliers of the pivot rows, unit diagonal
  double* rdiag;   // [n] IEEE 1 / U(t, t)
  unsigned long long* status;
  int n;
};
cudaError_t launch_tslu_leaf(int W, int64_t leaf_rows, const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                             const uint8_t* chosen, int* ids, int* cnt, double* vals, cudaStream_t st,
                             const RootOut* root = nullptr, unsigned long long* finite_status = nullptr);
// Candidate rows of a node: from the slot values (src == nullptr) or, on one process, straight
// from the panel source by global id: src + (id - row0) * lds + p0 (slots then carry ids only)
struct RowSrc {
  const double* src;
  int64_t lds, row0;
  int p0;
};
// vals may be null (ids-only slots) when the next level reads rows through a RowSrc
cudaError_t launch_tslu_node(int W, const int* in_ids, const int* in_cnt, const double* in_vals, int nin, int arity,
                             int w, int* ids, int* cnt, double* vals, cudaStream_t st, const RootOut* root = nullptr,
                             const RowSrc* rows = nullptr);
cudaError_t launch_tslu_panel_factor(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w, int n,
                                     const int* root_ids, const int* root_cnt, double* U, int64_t* piv,
                                     uint8_t* chosen, double* lpanel, unsigned long long* status, cudaStream_t st,
                                     int packed = 0);
cudaError_t launch_l11_fixup(double* L11, int n, cudaStream_t st);
cudaError_t launch_gather_rows(const double* src, int64_t lds, const int64_t* ids, int64_t row0, int cnt, int ncols,
                               double* dst, int64_t ldd, cudaStream_t st);
cudaError_t launch_pivpos(const int64_t* piv, int n, int64_t row0, int64_t rows, int* pivpos, cudaStream_t st);

// tslw.cu: warp-level tournament LU, left-looking 16-column panels (the default contract)
constexpr int kTslwPanel = 16;
struct TslwRoot {          // root outputs of one panel (all null below the root)
  double* U;               // n x n, ld n
  int64_t* piv;            // [n]
  double* rd;              // [n] 1 / U(t, t)
  double* lw;              // 16 x 16: in-panel multipliers of the panel's pivot rows
  uint8_t* chosen;         // local rows chosen as pivots
  unsigned long long* status;
  int64_t row0;
  int n;
};
// the warp kernels run this contract (tournament (128, <= 8, 16) or one leaf = exact GEPP)
bool tslw_cfg(const rlhc_tslu_cfg& c, int64_t m, int64_t n);
bool tslg_cfg(const rlhc_tslu_cfg& c, int64_t m, int64_t n);
size_t tslw_slots(int64_t rows);
// row-sharded local tree of the warp contract down to the slots of level stop_lev (-1: one
// slot, the local root) -- rlhc_tslu_reduce_to
cudaError_t run_tslw_local_tree(const double* src, int64_t lds, int64_t rows, int64_t row0, int p0, int w,
                                const uint8_t* chosen, int arity, int stop_lev, int* ids[2], int* cnt[2],
                                double* vals[2], int* out_ids, int* out_cnt, double* out_vals, cudaStream_t st);
cudaError_t run_tslw_schur_local_tree(const double* X, int64_t ldx, double* Lb, int64_t ldl, int64_t rows,
                                      int64_t row0, int p0, int w, int n, const double* U, const uint8_t* chosen,
                                      int arity, int stop_lev, int* ids[2], int* cnt[2], double* vals[2],
                                      int* out_ids, int* out_cnt, double* out_vals, unsigned long long* status,
                                      cudaStream_t st, bool* fused);
// rlhc_tslw_schur_reduce_to with the input check folded in (status, nullable); *checked: the
// panel's X columns were checked (false on the fallback path)
int tslw_schur_reduce_to_impl(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl,
                              int64_t row0, int64_t p0, const double* U, const uint8_t* chosen,
                              const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids, int* out_cnt,
                              double* out_vals, unsigned long long* status, bool* checked, void* ws, size_t ws_bytes,
                              cudaStream_t st);
// row-sharded left-looking TSLU blocks (the warp contract): a panel's Schur complement of
// this rank's rows (U's reciprocals from its diagonal), the winners' current rows this rank
// owns (0 for the others), and the last panel's L plus the local pivot rows' L11 rows
cudaError_t launch_tslw_schur(const double* X, int64_t ldx, double* Lb, int64_t ldl, int64_t rows, int p0, int w, int n,
                              const double* U, cudaStream_t st);
cudaError_t launch_tslw_owned(const double* X, int64_t ldx, const double* Lb, int64_t ldl, int64_t rows, int64_t row0,
                              const int* ids, int cnt, int p0, int n, const double* U, double* T, cudaStream_t st);
cudaError_t launch_tslw_finish(double* Lb, int64_t ldl, int64_t rows, int64_t row0, int n, const double* U,
                               const int64_t* piv, cudaStream_t st);
// exact GEPP mode (one leaf of all rows): workspace of the panel's working copy
size_t tslg_ws_bytes(int64_t rows);
// gepp_ws != null: exact GEPP (one leaf holding every row) instead of the tournament
// called by run_tslw right after each panel's Schur-complement launch (before its tournament):
// lets the caller put independent work on a side stream into the tournament's idle SMs
struct TslwPanelHook {
  cudaError_t (*after_schur)(void* ctx, int panel, int npanels, cudaStream_t st);
  void* ctx;
};
cudaError_t run_tslw(const double* X, int64_t ldx, int64_t rows, int64_t row0, int n, int arity, double* Lb,
                     int64_t ldl, int64_t* piv, double* U, double* L11, double* rd, double* lw, uint8_t* chosen,
                     int* ids[2], int* cnt[2], double* vals[2], unsigned long long* status, bool check_input,
                     cudaStream_t st, void* gepp_ws = nullptr, double* bpack = nullptr,
                     const TslwPanelHook* hook = nullptr);

// rows.cu
cudaError_t launch_check_finite(const double* X, int64_t rows, int n, int64_t ldx, unsigned long long* status,
                                cudaStream_t st);
cudaError_t launch_rdiag(const double* T, int n, int64_t ldt, double* rdiag, int stage, unsigned long long* status,
                         cudaStream_t st);
// out = A T^{-1} (substitution, fma chain in increasing k) on the first nsub columns,
// remaining columns [nsub, ncols) receive only the updates.  pivpos/L11: pivot-row override.
cudaError_t launch_trsm_rows(const double* A, int64_t lda, int64_t rows, int ncols, int nsub, const double* T,
                             int64_t ldt, const double* rdiag, double* out, int64_t ldo, const int* pivpos,
                             const double* L11, int64_t ldl11, cudaStream_t st);
// out = A Tinv (Tinv upper, full n x n storage with zero lower part); out may equal A.
cudaError_t launch_rows_upper(const double* A, int64_t lda, int64_t rows, int n, const double* Tinv, double* out,
                              int64_t ldo, cudaStream_t st);
size_t gram_partials_bytes(int64_t rows, int n);
size_t syrk_partials_bytes(int n);
cudaError_t launch_syrk(const double* A, int64_t lda, int64_t rows, int n, double* part, double* G, cudaStream_t st,
                        bool* done);
// fused persistent substitution (+ optional Gram of the output when G != nullptr), n <= 128
bool rowsolve_ok(int n);
size_t rowsolve_partials_bytes(int64_t rows, int n);
cudaError_t launch_rowsolve(const double* A, int64_t lda, int64_t rows, int n, const double* T, const double* rdiag,
                            double* out, int64_t ldo, const int64_t* piv, const double* L11, double* gpart, double* G,
                            cudaStream_t st);
// C_out = C_in - A B (rows x N, K <= 64) on DMMA, increasing-k chain
cudaError_t launch_gemm_update(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                               int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N, cudaStream_t st);
// blocked substitution for any n (rowsolve on 64-column panels + DMMA trailing updates)
cudaError_t launch_trsm_blocked(const double* A, int64_t lda, int64_t rows, int n, int nsub, const double* T,
                                int64_t ldt, const double* rdiag, double* out, int64_t ldo, cudaStream_t st);
cudaError_t launch_pivot_rows(const int64_t* piv, int n, int64_t row0, int64_t rows, const double* L11, double* out,
                              int64_t ldo, cudaStream_t st);
cudaError_t launch_gram(const double* A, int64_t lda, int64_t rows, int n, double* part, double* G, cudaStream_t st);
// out = A T^{-1} with the oracle's op sequence (separate multiply and subtract, IEEE
// division), n <= 64; out may alias A; G != null: G = out^T out fused (partials in gpart)
bool subst_ms_ok(int n);
size_t subst_ms_partials_bytes(int64_t rows, int n);
cudaError_t launch_subst_ms(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                            double* out, int64_t ldo, double* gpart, double* G, cudaStream_t st);

// sketch.cu
size_t gauss_partials_bytes(int64_t rows, int n, int s);
cudaError_t launch_sketch_gauss(const double* A, int64_t lda, int64_t rows, int n, int64_t row0, int s, uint64_t seed,
                                uint32_t stream_id, double* part, double* out, cudaStream_t st,
                                const double* Om = nullptr);
// Omega stored (s x cols, ld omega_ld(cols)) for the OMEM sketch; generated off the critical path
int64_t omega_ld(int64_t cols);
size_t omega_bytes(int64_t s, int64_t cols);
// columns [c0, c0 + ncols) of the s x m Omega (stream 0, global row ids) into Om (ld omega_ld(m))
cudaError_t launch_omega_gen_cols(uint64_t seed, int s, int64_t m, int64_t c0, int64_t ncols, double* Om,
                                  cudaStream_t st);
cudaError_t launch_omega_gen(uint64_t seed, uint32_t stream_id, int s, int64_t cols, int64_t row0, double* Om,
                             cudaStream_t st);
size_t cs_plan_bytes(int64_t rows, int s1);
cudaError_t launch_sketch_count(const double* A, int64_t lda, int64_t rows, int n, int64_t row0, int s1,
                                uint64_t seed, void* plan_ws, double* out, int32_t* bucket_out, int8_t* sign_out,
                                cudaStream_t st);
// the two halves of launch_sketch_count: the plan (hash, histogram, scan, scatter) depends
// only on the seed and sizes, so it can run off the critical path; apply gathers the buckets
cudaError_t launch_cs_plan(int64_t rows, int64_t row0, int s1, uint64_t seed, void* plan_ws, cudaStream_t st);
cudaError_t launch_cs_apply(const double* A, int64_t lda, int64_t rows, int n, int s1, void* plan_ws, double* out,
                            cudaStream_t st);

// small.cu
size_t hqr_ws_bytes(int s, int n);
cudaError_t launch_hqr(const double* A, int s, int n, int64_t lda, const double* sgn_ref, double* S, double* work,
                       unsigned long long* status, cudaStream_t st);
// R upper with R^T R = G; optionally 1/diag(R) (IEEE reciprocal, == rdiag_kernel's) into rdiag
cudaError_t launch_chol(const double* G, int n, double* R, double* work, int stage, unsigned long long* status,
                        cudaStream_t st, double* rdiag = nullptr);
size_t chol_ws_bytes(int n);
cudaError_t launch_tri_inv(const double* T, int n, double* Tinv, cudaStream_t st);
// tsgemm.cu: Cout = Cin -/+ A B on DMMA (persistent, TMA-fed, warp-specialised; the fma chain
// in increasing k); tri: B upper triangular, and Cout may then alias A (in-place triangular
// product).  bpack: ts_gemm_pack_bytes(K, N) bytes of scratch for B's packed image.
size_t ts_gemm_pack_bytes(int K, int N);
size_t tri_pack_bytes(int n);
cudaError_t launch_tri_tma(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int n, double* C,
                           int64_t ldc, double* bpack, cudaStream_t st, bool* done);
// launch_ts_gemm (tri = false, sub = true) that also reports a non-finite Cin element as
// ENONFINITE(INPUT, row * n_index + col0_index + column) into status (nullable)
cudaError_t launch_ts_gemm_checked(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A,
                                   int64_t lda, const double* B, int64_t ldb, int64_t rows, int K, int N, double* bpack,
                                   unsigned long long* status, int n_index, int col0_index, cudaStream_t st);
constexpr int kTslwGroup = 64;  // LU panels per bulk Schur product: 4 x 16 columns
// subst.cu: out = A T^{-1} in the oracle's operation order for n > 64 (W = X Y^-1, R#O9)
bool subst_wide_ok(int n);
cudaError_t launch_subst_wide(const double* A, int64_t lda, int64_t rows, int n, const double* T, int64_t ldt,
                              double* out, int64_t ldo, cudaStream_t st);
// the driver's cuTensorMapEncodeTiled (nullptr if unavailable); include <cudaTypedefs.h> to use
#ifdef PFN_cuTensorMapEncodeTiled
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
#endif
cudaError_t launch_ts_gemm(const double* Cin, int64_t ldci, double* Cout, int64_t ldco, const double* A, int64_t lda,
                           const double* B, int64_t ldb, int64_t rows, int K, int N, bool tri, bool sub, double* bpack,
                           cudaStream_t st);
cudaError_t launch_trmm_uu(const double* A, const double* B, int n, double* C, cudaStream_t st);
cudaError_t launch_shift_diag(double* G, int n, int64_t m, cudaStream_t st);
cudaError_t launch_flip_neg_rows(double* T, int n, cudaStream_t st);
cudaError_t launch_status_init(unsigned long long* status, cudaStream_t st);
cudaError_t launch_status_finish(const unsigned long long* status, void* info, cudaStream_t st);
cudaError_t launch_fill_i32(int* p, int64_t count, int value, cudaStream_t st);

}  // namespace rlhc
