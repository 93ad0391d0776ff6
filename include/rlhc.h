/*
 * rlhc.h -- C ABI of the B200 (sm_100a) hot path of randomized LU-Householder
 * CholeskyQR (rLHC), arXiv 2412.06551: SLHC3 (PAPER.md Algorithm alg:SLHC3,
 * P:301-311) and SSLHC3 (alg:SSLHC3) for tall-skinny fp64 X (m >> n).
 *
 * Conventions for every entry point
 *   - Matrices are IEEE fp64, ROW-major, with a leading dimension (ld >= number of
 *     columns).  Pointers named X, A, Q, R, U, L, G, S, T, out, ws are DEVICE pointers
 *     owned by the caller; nothing is allocated inside a call.
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default).
 *   - The int return value is host-side only: RLHC_OK, RLHC_EINVAL for an invalid
 *     argument (sizes, null pointers, leading dimensions, aliasing), RLHC_EWORKSPACE
 *     for a too-small workspace, RLHC_ECUDA for a launch failure (rlhc_last_error()
 *     gives the CUDA message).  Nothing is launched when the return value is not OK.
 *   - Numerical failures are written by the device into `info` (device pointer,
 *     first failure in pipeline order wins) and read by the caller after the stream
 *     is synchronised; outputs are unspecified when info->code != RLHC_OK.  Errors are
 *     values, never silent NaNs.
 *   - Inputs are never modified.  Results are bitwise reproducible for fixed inputs,
 *     seed, configuration and device (fixed-order reductions, no floating atomics).
 *   - Global row ids: `row0` is the global id of the first local row, so every
 *     random draw (Omega column, CountSketch hash) is indexed by the global row
 *     and row-sharded calls compose (R#2).
 */
#ifndef RLHC_H_
#define RLHC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rlhc_stream_t; /* == cudaStream_t */

/* Device-written status.  code: enum rlhc_code; stage: enum rlhc_stage; index:
 * the offending pivot / column / linear element index. */
typedef struct {
  int32_t code;
  int32_t stage;
  int64_t index;
} rlhc_info_t;

enum rlhc_code {
  RLHC_OK = 0,
  RLHC_EINVAL = 1,      /* host: invalid argument */
  RLHC_ENONFINITE = 2,  /* device: NaN/Inf in X (index = i*n + j) */
  RLHC_ERANKDEF = 3,    /* device: zero root pivot in PX = LU (index = k) or zero HQR column */
  RLHC_ESINGULAR = 4,   /* device: zero / non-finite diagonal of a triangular factor */
  RLHC_EBREAKDOWN = 5,  /* device: Cholesky pivot <= 0 or non-finite (index = k) */
  RLHC_ECUDA = 6,       /* host: CUDA launch error */
  RLHC_EWORKSPACE = 7,  /* host: workspace too small */
  RLHC_ENCCL = 8        /* host: NCCL unavailable or an NCCL call failed (_dist entry points) */
};

enum rlhc_stage {
  RLHC_STAGE_INPUT = 0,   /* finiteness of X */
  RLHC_STAGE_LU = 1,      /* PX = LU */
  RLHC_STAGE_SKETCH = 2,  /* L_s = Omega L / L_ss = Omega_2 Omega_1 L */
  RLHC_STAGE_HQR = 3,     /* [H, S] = HouseholderQR(L_s) */
  RLHC_STAGE_SOLVE_Y = 4, /* W = X Y^{-1}, Y = S U */
  RLHC_STAGE_CHOL1 = 5,   /* D = chol(W^T W) (P:27-28 inside CholeskyQR2) */
  RLHC_STAGE_SOLVE_D = 6, /* V = W D^{-1} */
  RLHC_STAGE_CHOL2 = 7,   /* J = chol(V^T V) */
  RLHC_STAGE_SOLVE_J = 8, /* Q = V J^{-1} */
  RLHC_STAGE_CHOL0 = 9,   /* the preconditioning Cholesky of the comparison methods (below) */
  RLHC_STAGE_COMM = 10    /* row-sharded calls: a replicated input differing across ranks
                             (RLHC_DIST_CHECK=1 debug check; code RLHC_ENCCL, index = count) */
};

enum rlhc_algo { RLHC_SLHC3 = 0, RLHC_SSLHC3 = 1 };
/* the paper's comparison algorithms, entry points below */
enum rlhc_method { RLHC_CHOLQR2 = 2, RLHC_SCHOLQR3 = 3, RLHC_LUC2 = 4, RLHC_RHC = 5 };
enum rlhc_trsm_mode { RLHC_SUBST = 0, RLHC_INV_GEMM = 1 };

/* Pivot-rule contract of PX = LU (R#3-R#5; the paper only says "P is a
 * permutation"): tournament pivoting over column panels of width `panel`
 * (panel = n is plain TSLU; a single leaf is GEPP).  Leaves are global row blocks
 * [l*leaf_rows, (l+1)*leaf_rows); each tree node runs GEPP on the stacked winners of
 * `arity` consecutive children (ties -> smallest global row id).  The result depends
 * only on (X, leaf_rows, arity, panel), never on the GPU count.  Supported on the
 * device: panel in {16, 32, 64} with leaf_rows == rows_per_select(panel) and
 * arity * panel <= rows_per_select(panel) (see rlhc_default_tslu_cfg). */
typedef struct {
  int64_t leaf_rows;
  int32_t arity;
  int32_t panel;
} rlhc_tslu_cfg;

/* Fills cfg with the device's default contract for an m x n problem (panel =
 * min(n rounded up to 16/32/64, 64), leaf_rows = candidate rows one select CTA
 * holds in registers, the largest arity that fits).  Never fails. */
void rlhc_default_tslu_cfg(int64_t m, int64_t n, rlhc_tslu_cfg* cfg);

/* Bytes of device workspace rlhc_slhc3 (algo = RLHC_SLHC3, s_or_s1 = s, s2 ignored) or
 * rlhc_sslhc3 (algo = RLHC_SSLHC3, s_or_s1 = s1, s2) needs; 0 on invalid sizes. */
size_t rlhc_workspace_size(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2, const rlhc_tslu_cfg* cfg);

/* SLHC3 (alg:SLHC3):  PX = LU; L_s = Omega L (Omega s x m Gaussian,
 * entries N(0, 1/s) from Philox stream 0, R#1/R#19); [H,S] =
 * HouseholderQR(L_s); Y = S U with sign(S_kk) = sign(U_kk) (R#7); W = X Y^{-1} by
 * substitution; [Q, Z] = CholeskyQR2(W); R = Z Y evaluated as J (D Y).
 *   X  : m x n, ldx >= n, rank n, m >= n, n <= s <= m.  Not modified.
 *   Q  : m x n output, ldq >= n; must not overlap X.  Used in place for L, W and V.
 *   R  : n x n output (row-major, strict lower part exactly 0, diag(R) > 0).
 *   piv: n int64 output, global row ids of the pivot rows in pivot order.
 *   ws : >= rlhc_workspace_size(RLHC_SLHC3, m, n, s, 0, cfg) bytes, 256-byte aligned.
 *   cfg: NULL = rlhc_default_tslu_cfg.  info: device pointer. */
int rlhc_slhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s, uint64_t seed,
               const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq, double* R, int64_t* piv, void* ws,
               size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);

/* SSLHC3 (alg:SSLHC3): as rlhc_slhc3 with L_ss = Omega_2 (Omega_1 L)
 * (P:294): Omega_1 s1 x m CountSketch (bucket/sign from Philox stream 2),
 * Omega_2 s2 x s1 Gaussian N(0, 1/s2) (stream 1).  n <= s2 <= s1 <= m. */
int rlhc_sslhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed,
                const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq, double* R, int64_t* piv, void* ws,
                size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);

/* ---------------------------------------------------------------- per-stage */
/* Row-pivoted tall-skinny LU "PX = LU" under the tslu contract.
 *   X: rows x n (rows = m, global ids row0..row0+rows-1; row0 must be 0 here).
 *   piv: n int64 out; U, L11: n x n out (U upper, L11 unit lower: multipliers of the
 *   pivot rows); L: nullable, rows x n out (ldl >= n), original row order.
 *   ws >= rlhc_getrf_ts_workspace_size(rows, n, cfg). */
size_t rlhc_getrf_ts_workspace_size(int64_t rows, int64_t n, const rlhc_tslu_cfg* cfg);
int rlhc_getrf_ts(const double* X, int64_t rows, int64_t n, int64_t ldx, int64_t row0, const rlhc_tslu_cfg* cfg,
                  int64_t* piv, double* U, double* L11, double* L, int64_t ldl, void* ws, size_t ws_bytes,
                  rlhc_info_t* info, rlhc_stream_t stream);

/* Gaussian sketch out (s x n, overwritten) = Omega A, where A is rows x n (lda) and
 * Omega's columns are the global rows row0..row0+rows-1: Omega[i, j] =
 * z_{i mod 2}(Philox(seed; j, i>>1, stream_id)) / sqrt(s) (R#19).
 * stream_id 0 = SLHC3's Omega, 1 = SSLHC3's Omega_2.  ws >= rlhc_sketch_gauss_workspace_size. */
size_t rlhc_sketch_gauss_workspace_size(int64_t rows, int64_t n, int64_t s);
int rlhc_sketch_gauss(const double* A, int64_t rows, int64_t n, int64_t lda, int64_t row0, int64_t s, uint64_t seed,
                      uint32_t stream_id, double* out, void* ws, size_t ws_bytes, rlhc_stream_t stream);

/* CountSketch out (s1 x n, overwritten) = Omega_1 A: global row j goes to
 * bucket(j) = (w0 * s1) >> 32 with sign (w1 >> 31 ? -1 : +1), (w0, w1) = Philox(seed;
 * j, 0, 2).  Each bucket is summed in ascending row order (deterministic).
 * bucket (int32[rows]) and sign (int8[rows]) are optional outputs (nullable). */
size_t rlhc_sketch_count_workspace_size(int64_t rows, int64_t n, int64_t s1);
int rlhc_sketch_count(const double* A, int64_t rows, int64_t n, int64_t lda, int64_t row0, int64_t s1, uint64_t seed,
                      double* out, int32_t* bucket, int8_t* sign, void* ws, size_t ws_bytes, rlhc_stream_t stream);

/* Gram G = A^T A, n x n full symmetric output (upper computed, mirrored:
 * exactly symmetric), split over rows with a fixed-order reduction. */
size_t rlhc_gram_workspace_size(int64_t rows, int64_t n);
int rlhc_gram(const double* A, int64_t rows, int64_t n, int64_t lda, double* G, void* ws, size_t ws_bytes,
              rlhc_stream_t stream);

/* out = A T^{-1} for n x n upper-triangular T ("Q = X R^{-1}").
 * mode RLHC_SUBST: row-wise substitution (backward stable for any kappa(T); used for
 * U and Y); for n <= 64 with the oracle's operation sequence per element (acc = a_k;
 * acc -= o_j T_jk as a rounded product then a rounded difference, j increasing; o_k =
 * acc / T_kk, IEEE division), for n > 64 blocked with the fma chain.  mode RLHC_INV_GEMM: T^{-1} formed once (n x n) then a streaming product
 * (used in the CholeskyQR2 tail where kappa(T) <= ~7).  out may equal A
 * (same pointer and ld: in place) but must not partially overlap it.  G_out: nullable
 * n x n, the Gram of out fused into the same pass.  A zero diagonal of T ->
 * ESINGULAR(SOLVE_Y, k) in info. */
size_t rlhc_trsm_apply_workspace_size(int64_t rows, int64_t n);
int rlhc_trsm_apply(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int mode, double* out,
                    int64_t ldo, double* G_out, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);

/* Householder R of an s x n matrix (LAPACK dgeqr2 order, H never formed):
 * S (n x n, upper) with the sign of row k flipped so sign(S_kk) = sign(sgn_ref_kk)
 * when sgn_ref (n x n, nullable) is given (R#7). A zero column -> ERANKDEF(HQR, k). */
size_t rlhc_hqr_workspace_size(int64_t s, int64_t n);
int rlhc_hqr_r(const double* A, int64_t s, int64_t n, int64_t lda, const double* sgn_ref, double* S, void* ws,
               size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);

/* Upper Cholesky factor of an n x n SPD matrix: pivot <= 0 or non-finite ->
 * EBREAKDOWN(stage, k) with the given stage tag. */
int rlhc_cholesky(const double* G, int64_t n, double* Rout, int stage, rlhc_info_t* info, rlhc_stream_t stream);

/* ------------------------------------------------- row-sharded (multi-GPU) building blocks */
/* SURVEY 8(e), DESIGN.md section 7.  Rank r holds global rows [row0, row0 + rows); the
 * orchestration (all-gather of tournament candidates, all-reduce of sketches / Grams /
 * pivot rows) is done by the caller (paper_2412_06551_b200/dist.py, torch.distributed);
 * every arithmetic step is one of these calls or a stage entry point above.
 * Tournament "slot" = (ids int32[W], cnt int32[1], vals double[W*W]) with W = 16/32/64 the
 * kernel width of cfg->panel: the winners of one tree node (global row ids in pivot
 * order, their current panel values row-major with stride W). */
size_t rlhc_tslu_local_workspace_size(int64_t rows, int64_t nslots_in, const rlhc_tslu_cfg* cfg);
/* leaves of this rank's rows + all local tree levels down to ONE slot (panel columns
 * [p0, p0 + w) of `src`; `chosen` (int8[rows], nullable) marks rows already pivots). */
int rlhc_tslu_reduce(const double* src, int64_t lds, int64_t rows, int64_t row0, int64_t p0, int64_t w,
                     const uint8_t* chosen, const rlhc_tslu_cfg* cfg, int* out_ids, int* out_cnt, double* out_vals,
                     void* ws, size_t ws_bytes, rlhc_stream_t stream);
/* the same down to `nslots_out` slots: the rank's rows are nslots_out complete subtrees of
 * the global tree (leaves / nslots_out a power of the arity), written as
 * consecutive slots out_ids[nslots_out * W], out_cnt[nslots_out], out_vals[nslots_out * W * W]
 * in global order.  RLHC_EINVAL when the leaf count does not split that way. */
int rlhc_tslu_reduce_to(const double* src, int64_t lds, int64_t rows, int64_t row0, int64_t p0, int64_t w,
                        const uint8_t* chosen, const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids,
                        int* out_cnt, double* out_vals, void* ws, size_t ws_bytes, rlhc_stream_t stream);
/* the number of slots a rank of `rows_local` rows reduces to under the contract: the leaf
 * count divided by the largest power of the arity dividing it (1 when it is a power). */
int64_t rlhc_tslu_local_slots(int64_t rows_local, const rlhc_tslu_cfg* cfg);
/* the tree levels above `nslots` consecutive slots (e.g. the all-gathered rank roots). */
int rlhc_tslu_combine(const int* in_ids, const int* in_cnt, const double* in_vals, int64_t nslots, int64_t w,
                      const rlhc_tslu_cfg* cfg, int* out_ids, int* out_cnt, double* out_vals, void* ws, size_t ws_bytes,
                      rlhc_stream_t stream);
/* out (w x ncols) = rows ids[t] (global, int32 or int64 list) of src, columns [c0, c0+ncols),
 * for the rows this rank owns, 0 otherwise (an all-reduce SUM then yields the rows exactly). */
int rlhc_owned_rows(const double* src, int64_t lds, int64_t rows, int64_t row0, const int* ids32, const int64_t* ids64,
                    int64_t w, int64_t c0, int64_t ncols, double* out, rlhc_stream_t stream);
/* U rows p0..p0+w-1 (columns p0..n-1) from the pivot rows `prow` (w x (n - p0), pivot order,
 * current values), piv[p0..), chosen[] of local pivot rows; zero pivot -> ERANKDEF(LU, k). */
size_t rlhc_tslu_panel_workspace_size(int64_t n);
int rlhc_tslu_panel_factor_rows(const double* prow, const int* ids, int64_t p0, int64_t w, int64_t n, int64_t row0,
                                int64_t rows, double* U, int64_t* piv, uint8_t* chosen, void* ws, size_t ws_bytes,
                                rlhc_info_t* info, rlhc_stream_t stream);
/* trailing update of this rank's rows with panel [p0, p0+w): dst[:, p0+w:] (dst may be src). */
size_t rlhc_tslu_eliminate_workspace_size(int64_t n);
int rlhc_tslu_eliminate(const double* src, int64_t lds, int64_t rows, int64_t p0, int64_t w, int64_t n,
                        const double* U, double* dst, int64_t ldd, void* ws, size_t ws_bytes, rlhc_stream_t stream);
/* L11 from the pivot rows of X (n x n, pivot order) and U; L of this rank's rows. */
/* Left-looking blocks of the warp contract (leaf_rows 128, 16-column panels; DESIGN.md
 * section 7), row-sharded: L is this rank's rows x n L buffer (the Q buffer).
 * rlhc_tslw_schur: panel [p0, p0+16) of this rank's rows.  p0 > 0: L's columns [p0-16, p0)
 *   (the previous panel's Schur values) become L by forward substitution with U's diagonal
 *   block; then L[:, p0:p0+w) = X[:, p0:p0+w) - L[:, :p0] U[:p0, p0:p0+w) (fma chain in
 *   increasing k, bit-identical to the single-process pipeline).  U: n x n, rows < p0 final.
 * rlhc_tslw_owned_rows: T (cnt x (n-p0), ld n-p0) = the current rows of the panel's winners
 *   ids[0..cnt) (global ids) over columns [p0, n) for the winners this rank owns, 0 for the
 *   others (an all-reduce sum gives every row exactly); input of rlhc_tslu_panel_factor_rows.
 * rlhc_tslw_finish: after the last panel: its Schur values become L, and this rank's pivot
 *   rows take their L11 rows (unit diagonal, zeros right of it).  L then equals the
 *   single-process rlhc_getrf_ts L rows of this rank.
 * All asynchronous on `stream`; EINVAL for bad sizes. */
int rlhc_tslw_schur(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl, int64_t p0,
                    const double* U, rlhc_stream_t stream);
/* rlhc_tslw_schur_reduce_to: rlhc_tslw_schur followed by rlhc_tslu_reduce_to(L, ...) on the
 *   panel just formed, fused as in the single-process pipeline: the leaves (128 of this rank's
 *   rows each, tournament of R#3) are selected inside the Schur kernel while it
 *   streams, then one launch runs this rank's levels >= 1 up to nslots_out complete subtrees
 *   (1: the rank's root).  Same outputs, bits and workspace (rlhc_tslu_local_workspace_size)
 *   as the two calls; falls back to them when X or L cannot be described to the TMA unit.
 *   chosen: this rank's rows already pivots (NULL at p0 = 0).  EINVAL unless the contract is
 *   the warp one (leaf_rows 128, panel 16, arity 2..8) and the leaves split into nslots_out
 *   complete subtrees; EWORKSPACE for a short workspace. */
int rlhc_tslw_schur_reduce_to(const double* X, int64_t rows, int64_t n, int64_t ldx, double* L, int64_t ldl,
                              int64_t row0, int64_t p0, const double* U, const uint8_t* chosen,
                              const rlhc_tslu_cfg* cfg, int64_t nslots_out, int* out_ids, int* out_cnt,
                              double* out_vals, void* ws, size_t ws_bytes, rlhc_stream_t stream);
int rlhc_tslw_owned_rows(const double* X, int64_t ldx, const double* L, int64_t ldl, int64_t rows, int64_t row0,
                         const int* ids, int64_t cnt, int64_t p0, int64_t n, const double* U, double* T,
                         rlhc_stream_t stream);
int rlhc_tslw_finish(double* L, int64_t ldl, int64_t rows, int64_t row0, int64_t n, const double* U,
                     const int64_t* piv, rlhc_stream_t stream);
size_t rlhc_lfactor_workspace_size(int64_t rows, int64_t n);
int rlhc_l11(const double* Xp, int64_t n, const double* U, double* L11, void* ws, size_t ws_bytes,
             rlhc_stream_t stream);
int rlhc_lfactor(const double* X, int64_t rows, int64_t n, int64_t ldx, int64_t row0, const double* U, const double* L11,
                 const int64_t* piv, double* L, int64_t ldl, void* ws, size_t ws_bytes, rlhc_stream_t stream);
/* C = A B for n x n upper-triangular A, B (zero lower parts); Cholesky with workspace (any n). */
int rlhc_trmm_upper(const double* A, const double* B, int64_t n, double* C, rlhc_stream_t stream);
size_t rlhc_cholesky_workspace_size(int64_t n);
int rlhc_cholesky_ws(const double* G, int64_t n, double* Rout, int stage, void* ws, size_t ws_bytes, rlhc_info_t* info,
                     rlhc_stream_t stream);

/* ------------------------------------------------- the paper's comparison algorithms */
/* The methods the paper compares SLHC3 / SSLHC3 against, on the same kernels (SURVEY 8(f)
 * NEXT-1; oracle: ora_cholqr2 / ora_scholqr3 / ora_luc2 / ora_rhc):
 *   rlhc_cholqr2   CholeskyQR2 (alg:cholqr2): [W,Y] = CholeskyQR(X), [Q,Z] =
 *                  CholeskyQR(W), R = Z Y;
 *   rlhc_scholqr3  SCholeskyQR3 (alg:Shifted3): shifted CholeskyQR with
 *                  s = 11 (m n u + (n+1) u) ||X||_g^2 (||X||_g = largest column norm,
 *                  DESIGN.md R#21), then CholeskyQR2;
 *   rlhc_luc2      LU-CholeskyQR2 (alg:LU2): PX = LU (tournament contract), S =
 *                  Cholesky(L^T L), Y = S U (diag > 0, R#23), W = X Y^{-1}, CholeskyQR(W);
 *   rlhc_rhc       Rand.Householder-Cholesky (alg:Rand2): K = Omega_2 Omega_1 X
 *                  (CountSketch s1 + Gaussian s2, the SSLHC3 streams), Y = HouseholderQR(K)
 *                  (diag > 0, R#22), W = X Y^{-1}, CholeskyQR(W).
 * Same conventions as rlhc_slhc3: device pointers, row-major, Q (m x n) must not alias X,
 * R (n x n, strict lower 0, diag > 0), info = first device error (breakdown of the first
 * Cholesky: EBREAKDOWN(RLHC_STAGE_CHOL0, k); of the CholeskyQR tail: CHOL1 / CHOL2). */
size_t rlhc_method_workspace_size(int method, int64_t m, int64_t n, int64_t s1, int64_t s2,
                                  const rlhc_tslu_cfg* cfg);
int rlhc_cholqr2(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R, void* ws,
                 size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);
int rlhc_scholqr3(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R, void* ws,
                  size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);
int rlhc_luc2(const double* X, int64_t m, int64_t n, int64_t ldx, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq,
              double* R, int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);
int rlhc_rhc(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed, double* Q,
             int64_t ldq, double* R, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_stream_t stream);

/* ------------------------------------------------- row-sharded entry points over NCCL */
/* SURVEY 8(b) "_dist", 8(e).  The whole SLHC3 / SSLHC3 call on nranks GPUs, one process per
 * GPU, orchestrated in C on the caller's stream (no host synchronisation): TSLU candidates
 * all-gathered, pivot rows / sketches / Grams all-reduced (NCCL, SUM), the n x n factors
 * replicated; DESIGN.md section 7.  NCCL is loaded at run time (dlopen "libnccl.so.2").
 * Communicator: rank 0 calls rlhc_comm_unique_id (128 bytes), the caller distributes the
 * bytes (e.g. torch.distributed), every rank calls rlhc_comm_init; nullptr = one rank.
 * Shards: equal, rank r holds global rows [row0, row0 + m_local), row0 = r * m_local,
 * m_local a multiple of cfg->leaf_rows and (nranks > 1) m_local / leaf_rows a power of
 * cfg->arity, so the pivots are those of the single-GPU tournament on the whole X.
 * Outputs: Q (m_local x n, this rank's rows), R (n x n, replicated), piv (n, global ids,
 * replicated); info: the first device error in pipeline order (same codes / stages as the
 * single-GPU call).  Errors: host argument checks -> RLHC_EINVAL / RLHC_EWORKSPACE,
 * NCCL failures -> RLHC_ENCCL (message in rlhc_last_error). */
typedef struct rlhc_comm_s* rlhc_comm_t;
int rlhc_comm_unique_id(void* id_out /* 128 bytes */);
int rlhc_comm_init(rlhc_comm_t* comm, int nranks, int rank, const void* id /* 128 bytes */);
int rlhc_comm_destroy(rlhc_comm_t comm);
size_t rlhc_dist_workspace_size(int algo, int64_t m_local, int64_t n, int64_t s_or_s1, int64_t s2,
                                const rlhc_tslu_cfg* cfg, int nranks);
int rlhc_slhc3_dist(const double* X, int64_t m_local, int64_t n, int64_t ldx, int64_t row0, int64_t m_global,
                    int64_t s, uint64_t seed, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq, double* R,
                    int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_comm_t comm,
                    rlhc_stream_t stream);
int rlhc_sslhc3_dist(const double* X, int64_t m_local, int64_t n, int64_t ldx, int64_t row0, int64_t m_global,
                     int64_t s1, int64_t s2, uint64_t seed, const rlhc_tslu_cfg* cfg, double* Q, int64_t ldq,
                     double* R, int64_t* piv, void* ws, size_t ws_bytes, rlhc_info_t* info, rlhc_comm_t comm,
                     rlhc_stream_t stream);

/* Library identification and the last host-side error message (thread-local). */
const char* rlhc_version(void);
const char* rlhc_last_error(void);

/* ---------------------------------------------------------------- CUDA graphs */
/* ---- Host-buffer pipeline (end to end through the C ABI).
 * `count` independent problems of one shape, inputs and outputs in HOST memory: problem i
 * factors X_host[i] (m x n, row-major, ld n) with seed seeds[i] by SLHC3 (algo RLHC_SLHC3,
 * s_or_s1 = s) or SSLHC3 (RLHC_SSLHC3, s_or_s1 = s1, s2) exactly as
 * rlhc_slhc3 / rlhc_sslhc3 do, and writes Q_host[i] (m x n, ld n), R_host[i] (n x n),
 * piv_host[i] (n int64, the array or an entry may be NULL) and info_host[i].
 * Device copies are double-buffered inside `ws`: the host->device copy of problem i+1 and the
 * device->host copies of problem i-1 run on two library-internal copy streams while problem i
 * computes on `stream`.  Host buffers (info_host and piv_host included) should be pinned
 * (cudaHostAlloc / cudaHostRegister): a copy into pageable memory blocks the enqueueing thread.  The call only enqueues; `stream` completes after the last copy, so
 * synchronise it before reading the host outputs.  ws: device memory of
 * rlhc_host_pipeline_workspace_size bytes, 256-byte aligned, owned by the caller, not to be
 * used concurrently by another call.  Errors: RLHC_EINVAL (sizes, pointers, configuration),
 * RLHC_EWORKSPACE, RLHC_ECUDA; numerical outcomes per problem in info_host[i]. */
size_t rlhc_host_pipeline_workspace_size(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2,
                                         const rlhc_tslu_cfg* cfg);
int rlhc_host_pipeline(int algo, int64_t count, const double* const* X_host, int64_t m, int64_t n, int64_t s_or_s1,
                       int64_t s2, const uint64_t* seeds, const rlhc_tslu_cfg* cfg, double* const* Q_host,
                       double* const* R_host, int64_t* const* piv_host, rlhc_info_t* info_host, void* ws,
                       size_t ws_bytes, rlhc_stream_t stream);

/* Launch-latency cut for small problems: capture one
 * stream-ordered call (rlhc_slhc3, rlhc_sslhc3, a comparison method, a stage entry point)
 * into a CUDA graph and replay it.  rlhc_graph_begin(stream) starts a thread-local
 * capture on `stream` (which must not be the legacy default stream); the calls issued on
 * it are recorded, not run; rlhc_graph_end(stream, &g) instantiates the graph.
 * rlhc_graph_launch(g, stream) replays it: the same kernels on the same pointers (the
 * CONTENTS of X may change between replays; sizes, pointers and workspace may not).
 * Stage timing is suspended while capturing.  Returns RLHC_OK, RLHC_EINVAL (null / no
 * capture in progress) or RLHC_ECUDA (rlhc_last_error has the CUDA message; a failed
 * end discards the capture). */
typedef struct rlhc_graph_s* rlhc_graph_t;
int rlhc_graph_begin(rlhc_stream_t stream);
int rlhc_graph_end(rlhc_stream_t stream, rlhc_graph_t* graph);
int rlhc_graph_launch(rlhc_graph_t graph, rlhc_stream_t stream);
void rlhc_graph_destroy(rlhc_graph_t graph);

/* ---------------------------------------------------------------- diagnostics */
/* Number of CUDA kernels this library has launched in the calling process. */
uint64_t rlhc_launch_count(void);
/* enable != 0: rlhc_slhc3 / rlhc_sslhc3 record a CUDA event on their stream at every
 * stage boundary (RLHC_NUM_TIMED_STAGES stages, see rlhc_stage_name); 0 disables and
 * discards pending events. */
void rlhc_stage_timing(int enable);
/* Synchronises the recorded events, adds each stage's elapsed milliseconds to ms[k]
 * (k < max_stages), returns the number of calls consumed (or -1 on a CUDA error). */
int rlhc_stage_times(double* ms, int max_stages);
const char* rlhc_stage_name(int k);
#define RLHC_NUM_TIMED_STAGES 13

#ifdef __cplusplus
}
#endif
#endif /* RLHC_H_ */
