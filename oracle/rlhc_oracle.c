/*
 * rlhc_oracle.c -- plain, slow, obviously-correct CPU fp64 oracle for the hot
 * path of randomized LU-Householder CholeskyQR (SLHC3 / SSLHC3), arXiv 2412.06551.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2412_06551_b200/).
 *
 * Citations: "P:n" = PAPER.md line n (LaTeX source of the paper), "R#k" = the
 * k-th reading of the paper listed in DESIGN.md section 3 (where the paper is
 * silent or garbled).  Each function states the passage it follows.
 *
 * Compile: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no contraction: every
 * fused multiply-add below is an explicit fma()).
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py against
 * the paper's worked examples, closed forms, LAPACK / numpy, brute force or
 * invariants.  Parity unpinned: none.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ errors */
/* Error model: errors are values, stage-tagged. */
enum { ORA_OK = 0, ORA_EINVAL = 1, ORA_ENONFINITE = 2, ORA_ERANKDEF = 3, ORA_ESINGULAR = 4, ORA_EBREAKDOWN = 5 };
enum { ST_INPUT = 0, ST_LU = 1, ST_SKETCH = 2, ST_HQR = 3, ST_SOLVE_Y = 4, ST_CHOL1 = 5, ST_SOLVE_D = 6,
       ST_CHOL2 = 7, ST_SOLVE_J = 8, ST_CHOL0 = 9 };
typedef struct { int32_t code; int32_t stage; int64_t index; } ora_info;

static int set_err(ora_info* info, int code, int stage, int64_t index) {
  if (info) { info->code = code; info->stage = stage; info->index = index; }
  return code;
}

/* ---------------------------------------------------------------- Philox */
/* Philox4x32-10 (Salmon et al., SC'11) -- the counter-based generator that defines
 * Omega, Omega_2 and the CountSketch hash (R#19: the paper gives no RNG). */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
  c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void ora_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; r++) {
    if (r) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
    philox_round(c, k);
  }
  memcpy(out, c, sizeof c);
}

/* counter = (j lo, j hi, c2, stream), key = (seed lo, seed hi)  (R#19) */
static void philox_words(uint64_t seed, uint64_t j, uint32_t c2, uint32_t stream, uint32_t w[4]) {
  uint32_t ctr[4] = {(uint32_t)j, (uint32_t)(j >> 32), c2, stream};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  ora_philox(ctr, key, w);
}

/* ------------------------------------------------- deterministic log / sincos */
/* The Gaussian transform (R#19) is defined by a fixed operation sequence so
 * that any IEEE-754 implementation reproduces it bit for bit:
 *   log x  = e*ln2 + 2t * sum_{k=0}^{11} t^{2k}/(2k+1),  t = (f-1)/(f+1),
 *            x = f*2^e with f in (sqrt2/2, sqrt2]
 *   sin/cos(2*pi*u): q = floor(4u + 1/2), r = 4u - q, theta = r*pi/2, Taylor
 *            series to theta^19 / theta^18, quadrant swap by q mod 4.
 * Coefficients are computed as IEEE quotients 1/(2k+1) and 1/k! (k! exact). */
static double c_log[12], c_sin[10], c_cos[10];
static const double LN2_HI = 0x1.62e42fefa39efp-1, LN2_LO = 0x1.abc9e3b39803fp-56;
static const double SQRT2 = 0x1.6a09e667f3bcdp+0;
static const double PIO2_HI = 0x1.921fb54442d18p+0, PIO2_LO = 0x1.1a62633145c07p-54;

__attribute__((constructor)) static void init_coeffs(void) {
  for (int k = 0; k < 12; k++) c_log[k] = 1.0 / (double)(2 * k + 1);
  double f = 1.0; /* running factorial, exact up to 22! */
  double fact[20];
  fact[0] = 1.0;
  for (int k = 1; k < 20; k++) { f = f * (double)k; fact[k] = f; }
  for (int k = 0; k < 10; k++) {
    double sgn = (k & 1) ? -1.0 : 1.0;
    c_sin[k] = sgn * (1.0 / fact[2 * k + 1]); /* (-1)^k/(2k+1)! */
    c_cos[k] = sgn * (1.0 / fact[2 * k]);     /* (-1)^k/(2k)!   */
  }
}

double ora_det_log(double x) { /* x > 0, normal */
  uint64_t b; memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  uint64_t fb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double f; memcpy(&f, &fb, 8);
  if (f > SQRT2) { f = f * 0.5; e += 1; }
  double t = (f - 1.0) / (f + 1.0);
  double t2 = t * t;
  double p = c_log[11];
  for (int k = 10; k >= 0; k--) p = fma(p, t2, c_log[k]);
  double lf = (2.0 * t) * p;
  double de = (double)e;
  return fma(de, LN2_HI, fma(de, LN2_LO, lf));
}

void ora_det_sincos2pi(double u, double* s_out, double* c_out) { /* u in [0,1) */
  double x = 4.0 * u;
  int64_t q = (int64_t)(x + 0.5);
  double r = x - (double)q;
  double th = fma(r, PIO2_HI, r * PIO2_LO);
  double t2 = th * th;
  double sp = c_sin[9];
  for (int k = 8; k >= 1; k--) sp = fma(sp, t2, c_sin[k]);
  double sn = fma(th * t2, sp, th);
  double cp = c_cos[9];
  for (int k = 8; k >= 1; k--) cp = fma(cp, t2, c_cos[k]);
  double cs = fma(t2, cp, 1.0);
  switch (q & 3) {
    case 0: *s_out = sn; *c_out = cs; break;
    case 1: *s_out = cs; *c_out = -sn; break;
    case 2: *s_out = -sn; *c_out = -cs; break;
    default: *s_out = -cs; *c_out = sn; break;
  }
}

/* Box-Muller pair from one Philox block (R#19):
 *   u1 = ((w1:w0) >> 11 + 1) 2^-53 in (0,1],  u2 = ((w3:w2) >> 11) 2^-53 in [0,1)
 *   z0 = sqrt(-2 log u1) cos(2 pi u2),  z1 = sqrt(-2 log u1) sin(2 pi u2). */
void ora_gauss_pair(uint64_t seed, uint64_t j, uint32_t c2, uint32_t stream, double* z0, double* z1) {
  uint32_t w[4];
  philox_words(seed, j, c2, stream, w);
  uint64_t a = ((((uint64_t)w[1]) << 32) | w[0]) >> 11;
  uint64_t b = ((((uint64_t)w[3]) << 32) | w[2]) >> 11;
  double u1 = (double)(a + 1) * 0x1p-53;
  double u2 = (double)b * 0x1p-53;
  double r = sqrt(-2.0 * ora_det_log(u1));
  double sn, cs;
  ora_det_sincos2pi(u2, &sn, &cs);
  *z0 = r * cs;
  *z1 = r * sn;
}

/* Gaussian sketch entry ("Omega = (1/s) G" read as N(0,1/s), R#1):
 * Omega[i,j] = z_{i mod 2}(counter = (j, i>>1, stream)) * (1/sqrt(s)). */
double ora_omega(uint64_t seed, uint32_t stream, int64_t s, int64_t i, int64_t j) {
  double z0, z1;
  ora_gauss_pair(seed, (uint64_t)j, (uint32_t)(i >> 1), stream, &z0, &z1);
  double sc = 1.0 / sqrt((double)s);
  return ((i & 1) ? z1 : z0) * sc;
}

/* dense s x cols block of Omega for columns j0..j0+cols-1 (test helper) */
void ora_omega_block(uint64_t seed, uint32_t stream, int64_t s, int64_t j0, int64_t cols, double* out) {
  for (int64_t i = 0; i < s; i++)
    for (int64_t c = 0; c < cols; c++) out[i * cols + c] = ora_omega(seed, stream, s, i, j0 + c);
}

/* ------------------------------------------------------------- CountSketch */
/* CountSketch Omega_1: one +-1 per column j of
 * Omega_1 (= row j of L).  Hash (R#19): Philox words of counter (j, 0, 0, 2):
 * bucket = (w0 * s1) >> 32, sign = (w1 >> 31) ? -1 : +1. */
void ora_cs_hash(uint64_t seed, int64_t row0, int64_t rows, int64_t s1, int32_t* bucket, int8_t* sign) {
  for (int64_t r = 0; r < rows; r++) {
    uint32_t w[4];
    philox_words(seed, (uint64_t)(row0 + r), 0u, 2u, w);
    bucket[r] = (int32_t)(((uint64_t)w[0] * (uint64_t)s1) >> 32);
    sign[r] = (w[1] >> 31) ? (int8_t)-1 : (int8_t)1;
  }
}

/* out (s1 x n) = Omega_1 A, Omega_1[bucket[j], j] = sign[j];
 * accumulation in ascending j. */
void ora_cs_apply(const double* A, int64_t rows, int64_t n, int64_t lda, const int32_t* bucket,
                  const int8_t* sign, int64_t s1, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(s1 * n));
  for (int64_t j = 0; j < rows; j++) {
    double* o = out + (int64_t)bucket[j] * n;
    const double* a = A + j * lda;
    if (sign[j] > 0) for (int64_t c = 0; c < n; c++) o[c] += a[c];
    else             for (int64_t c = 0; c < n; c++) o[c] -= a[c];
  }
}

/* out (s x n) = Omega A with Omega's columns row0..row0+rows-1;
 * sum over rows in ascending j, fixed 64-chunk partition for OpenMP (deterministic). */
void ora_sketch_gauss(const double* A, int64_t rows, int64_t n, int64_t lda, int64_t row0, int64_t s,
                      uint64_t seed, uint32_t stream, double* out) {
  const int NCH = 64;
  double* part = (double*)calloc((size_t)NCH * s * n, sizeof(double));
  #pragma omp parallel for schedule(static)
  for (int ch = 0; ch < NCH; ch++) {
    int64_t a0 = rows * ch / NCH, a1 = rows * (ch + 1) / NCH;
    double* P = part + (size_t)ch * s * n;
    double* om = (double*)malloc(sizeof(double) * (size_t)s);
    for (int64_t j = a0; j < a1; j++) {
      for (int64_t i = 0; i < s; i += 2) {
        double z0, z1;
        ora_gauss_pair(seed, (uint64_t)(row0 + j), (uint32_t)(i >> 1), stream, &z0, &z1);
        double sc = 1.0 / sqrt((double)s);
        om[i] = z0 * sc;
        if (i + 1 < s) om[i + 1] = z1 * sc;
      }
      const double* a = A + j * lda;
      for (int64_t i = 0; i < s; i++) {
        double w = om[i];
        double* p = P + i * n;
        for (int64_t c = 0; c < n; c++) p[c] += w * a[c];
      }
    }
    free(om);
  }
  memset(out, 0, sizeof(double) * (size_t)(s * n));
  for (int ch = 0; ch < NCH; ch++)
    for (int64_t t = 0; t < s * n; t++) out[t] += part[(size_t)ch * s * n + t];
  free(part);
}

/* ---------------------------------------------------------------- TSLU */
/* Tournament pivot selection (R#3, R#4, R#5): GEPP on `cnt` candidate rows
 * (values B, cnt x w row-major, ids = global row ids).  For t = 0..min(cnt,w)-1:
 * p = argmax |B[i,t]| over remaining rows, ties -> smallest id; if that maximum
 * is 0 the remaining row with the smallest id is taken and nothing is updated;
 * otherwise r = 1/B[p,t], l = B[i,t]*r, B[i,j] = fma(-l, B[p,j], B[i,j]) (j>t).
 * B is overwritten.  Returns the number of selected rows. */
static int64_t gepp_select(double* B, const int64_t* ids, int64_t cnt, int64_t w, int64_t* out_ids) {
  char* done = (char*)calloc((size_t)(cnt > 0 ? cnt : 1), 1);
  int64_t steps = cnt < w ? cnt : w;
  for (int64_t t = 0; t < steps; t++) {
    int64_t p = -1; double best = -1.0;
    for (int64_t i = 0; i < cnt; i++) {
      if (done[i]) continue;
      double v = fabs(B[i * w + t]);
      if (p < 0 || v > best || (v == best && ids[i] < ids[p])) { p = i; best = v; }
    }
    if (p < 0) break;
    if (best == 0.0) { /* zero column: smallest remaining id, no update (R#5) */
      p = -1;
      for (int64_t i = 0; i < cnt; i++) if (!done[i] && (p < 0 || ids[i] < ids[p])) p = i;
      done[p] = 1; out_ids[t] = ids[p];
      continue;
    }
    done[p] = 1; out_ids[t] = ids[p];
    double r = 1.0 / B[p * w + t];
    for (int64_t i = 0; i < cnt; i++) {
      if (done[i]) continue;
      double l = B[i * w + t] * r;
      B[i * w + t] = l;
      for (int64_t j = t + 1; j < w; j++) B[i * w + j] = fma(-l, B[p * w + j], B[i * w + j]);
    }
  }
  free(done);
  return steps;
}

/* Row-pivoted LU "PX = LU" with tournament pivoting over
 * column panels of width `panel` (R#3; panel = n is plain TSLU, one leaf is GEPP).
 * For each panel [p0, p0+w): leaves are global row blocks [l*b, (l+1)*b) of the
 * rows not yet chosen as pivots; a node groups `arity` consecutive children and
 * runs gepp_select on the stacked winners (current values of the panel columns);
 * the root's winners are this panel's pivots, in pivot order.  Then every
 * remaining row is eliminated with those pivots (same fma chain as in the select):
 *   A[i,k] <- l = A[i,k] * (1/U[k,k]);  A[i,j] <- fma(-l, U[k,j], A[i,j]), j > k.
 * Outputs: piv (pivot order), U (n x n upper, row k = pivot row k), L11 (n x n
 * unit lower: multipliers of the pivot rows), optionally L (m x n, original row
 * order).  A zero pivot at the root -> ERANKDEF(LU, k). */
int ora_tslu(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t b, int64_t arity, int64_t panel,
             int64_t* piv, double* U, double* L11, double* L, ora_info* info) {
  if (m < n || n < 1 || b < 1 || arity < 2 || panel < 1 || ldx < n) return set_err(info, ORA_EINVAL, ST_LU, 0);
  double* A = (double*)malloc(sizeof(double) * (size_t)(m * n));
  for (int64_t i = 0; i < m; i++) memcpy(A + i * n, X + i * ldx, sizeof(double) * (size_t)n);
  char* chosen = (char*)calloc((size_t)m, 1);
  int64_t nleaves = (m + b - 1) / b;
  int rc = ORA_OK;
  for (int64_t p0 = 0; p0 < n && rc == ORA_OK; p0 += panel) {
    int64_t w = (n - p0) < panel ? (n - p0) : panel;
    /* level 0: leaves */
    int64_t nn = nleaves;
    int64_t* cnt = (int64_t*)calloc((size_t)nn, sizeof(int64_t));
    int64_t* win = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nn * w));
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t l = 0; l < nleaves; l++) {
      int64_t r0 = l * b, r1 = (r0 + b < m) ? r0 + b : m;
      int64_t c = 0;
      int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r1 - r0));
      double* B = (double*)malloc(sizeof(double) * (size_t)((r1 - r0) * w));
      for (int64_t i = r0; i < r1; i++) {
        if (chosen[i]) continue;
        ids[c] = i;
        memcpy(B + c * w, A + i * n + p0, sizeof(double) * (size_t)w);
        c++;
      }
      cnt[l] = gepp_select(B, ids, c, w, win + l * w);
      free(ids); free(B);
    }
    /* internal levels */
    while (nn > 1) {
      int64_t np = (nn + arity - 1) / arity;
      int64_t* cnt2 = (int64_t*)calloc((size_t)np, sizeof(int64_t));
      int64_t* win2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(np * w));
      #pragma omp parallel for schedule(dynamic, 1)
      for (int64_t t = 0; t < np; t++) {
        int64_t c0 = t * arity, c1 = (c0 + arity < nn) ? c0 + arity : nn;
        int64_t tot = 0;
        for (int64_t c = c0; c < c1; c++) tot += cnt[c];
        int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(tot > 0 ? tot : 1));
        double* B = (double*)malloc(sizeof(double) * (size_t)((tot > 0 ? tot : 1) * w));
        int64_t q = 0;
        for (int64_t c = c0; c < c1; c++)
          for (int64_t e = 0; e < cnt[c]; e++) {
            ids[q] = win[c * w + e];
            memcpy(B + q * w, A + ids[q] * n + p0, sizeof(double) * (size_t)w);
            q++;
          }
        cnt2[t] = gepp_select(B, ids, tot, w, win2 + t * w);
        free(ids); free(B);
      }
      free(cnt); free(win);
      cnt = cnt2; win = win2; nn = np;
    }
    if (cnt[0] < w) { rc = set_err(info, ORA_ERANKDEF, ST_LU, p0 + cnt[0]); free(cnt); free(win); break; }
    for (int64_t t = 0; t < w; t++) piv[p0 + t] = win[t];
    free(cnt); free(win);
    /* elimination of the remaining rows with this panel's pivots */
    for (int64_t k = p0; k < p0 + w; k++) {
      int64_t p = piv[k];
      chosen[p] = 1;
      double ukk = A[p * n + k];
      if (ukk == 0.0) { rc = set_err(info, ORA_ERANKDEF, ST_LU, k); break; }
      double r = 1.0 / ukk;
      const double* up = A + p * n;
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < m; i++) {
        if (chosen[i]) continue;
        double* a = A + i * n;
        double l = a[k] * r;
        a[k] = l;
        for (int64_t j = k + 1; j < n; j++) a[j] = fma(-l, up[j], a[j]);
      }
    }
  }
  if (rc == ORA_OK) {
    memset(U, 0, sizeof(double) * (size_t)(n * n));
    memset(L11, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t k = 0; k < n; k++) {
      const double* a = A + piv[k] * n;
      for (int64_t j = k; j < n; j++) U[k * n + j] = a[j];
      for (int64_t j = 0; j < k; j++) L11[k * n + j] = a[j];
      L11[k * n + k] = 1.0;
    }
    if (L) {
      for (int64_t i = 0; i < m; i++) memcpy(L + i * n, A + i * n, sizeof(double) * (size_t)n);
      for (int64_t k = 0; k < n; k++) memcpy(L + piv[k] * n, L11 + k * n, sizeof(double) * (size_t)n);
    }
  }
  free(A); free(chosen);
  return rc;
}

/* Row j of L in original order (R#2): a pivot row takes its L11 row;
 * any other row solves l U = x by forward substitution with the same fma chain
 * as the elimination: acc = x_k; acc = fma(-l_k', U[k',k], acc) for k' < k;
 * l_k = acc * (1/U[k,k]).  pivpos[j] = k if j = piv[k], else -1. */
static void l_row(const double* x, int64_t n, const double* U, const double* rdiag, const double* L11,
                  int64_t pp, double* l) {
  if (pp >= 0) { memcpy(l, L11 + pp * n, sizeof(double) * (size_t)n); return; }
  for (int64_t k = 0; k < n; k++) {
    double acc = x[k];
    for (int64_t kk = 0; kk < k; kk++) acc = fma(-l[kk], U[kk * n + k], acc);
    l[k] = acc * rdiag[k];
  }
}

int64_t* ora_pivpos(const int64_t* piv, int64_t m, int64_t n) {
  int64_t* pp = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  for (int64_t i = 0; i < m; i++) pp[i] = -1;
  for (int64_t k = 0; k < n; k++) pp[piv[k]] = k;
  return pp;
}

/* full L (m x n) from X, piv, U, L11 by row substitution (test helper) */
void ora_lfactor(const double* X, int64_t m, int64_t n, int64_t ldx, const int64_t* piv, const double* U,
                 const double* L11, double* L) {
  int64_t* pp = ora_pivpos(piv, m, n);
  double* rd = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t k = 0; k < n; k++) rd[k] = 1.0 / U[k * n + k];
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) l_row(X + i * ldx, n, U, rd, L11, pp[i], L + i * n);
  free(rd); free(pp);
}

/* ------------------------------------------------------------ dense kernels */
/* Householder QR, only R kept (Lemma 2.3), unblocked in
 * LAPACK dgeqr2 order: beta = -sign(alpha) ||x||_2 (sign(0) = +1), tau = (beta-alpha)/beta,
 * v = x(2:)/(alpha-beta), A(k:,k+1:) -= tau v (v^T A(k:,k+1:)).  A zero column
 * -> ERANKDEF(HQR, k).  A (s x n) is overwritten; R = its upper n x n part. */
static double nrm2_scaled(const double* x, int64_t cnt, int64_t stride) {
  double scale = 0.0;
  for (int64_t i = 0; i < cnt; i++) { double a = fabs(x[i * stride]); if (a > scale) scale = a; }
  if (scale == 0.0) return 0.0;
  double ssq = 0.0;
  for (int64_t i = 0; i < cnt; i++) { double t = x[i * stride] / scale; ssq += t * t; }
  return scale * sqrt(ssq);
}

int ora_hqr_r(double* A, int64_t s, int64_t n, double* R, ora_info* info) {
  if (s < n) return set_err(info, ORA_EINVAL, ST_HQR, 0);
  double* wv = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t k = 0; k < n; k++) {
    double alpha = A[k * n + k];
    double xnorm = nrm2_scaled(A + (k + 1) * n + k, s - k - 1, n);
    if (xnorm == 0.0 && alpha == 0.0) { free(wv); return set_err(info, ORA_ERANKDEF, ST_HQR, k); }
    if (xnorm == 0.0) continue; /* H = I, tau = 0 */
    double beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, xnorm);
    double tau = (beta - alpha) / beta;
    double sc = 1.0 / (alpha - beta);
    for (int64_t i = k + 1; i < s; i++) A[i * n + k] *= sc; /* v, v_0 = 1 */
    A[k * n + k] = beta;
    for (int64_t j = k + 1; j < n; j++) {
      double w = A[k * n + j];
      for (int64_t i = k + 1; i < s; i++) w += A[i * n + k] * A[i * n + j];
      wv[j] = w;
    }
    for (int64_t j = k + 1; j < n; j++) {
      double tw = tau * wv[j];
      A[k * n + j] -= tw;
      for (int64_t i = k + 1; i < s; i++) A[i * n + j] -= A[i * n + k] * tw;
    }
  }
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = 0; j < n; j++) R[i * n + j] = (j >= i) ? A[i * n + j] : 0.0;
  free(wv);
  return ORA_OK;
}

/* C = A B for n x n upper-triangular A, B (R = SU P:282, N = DY P:711, R = JN P:715);
 * C[i,j] = sum_{k=i..j} A[i,k] B[k,j]; strict lower part exactly 0. */
void ora_trmm_uu(const double* A, const double* B, int64_t n, double* C) {
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = 0; j < n; j++) {
      double acc = 0.0;
      if (j >= i) for (int64_t k = i; k <= j; k++) acc += A[i * n + k] * B[k * n + j];
      C[i * n + j] = acc;
    }
}

/* out = A T^{-1} for n x n upper T by row-wise substitution, never forming T^{-1}
 * ("Q = X R^{-1}"): out_k = (a_k - sum_{k'<k} out_k' T[k',k]) / T[k,k].
 * A zero or non-finite diagonal -> ESINGULAR(stage, k).  out may alias A (row by row). */
int ora_trsm_right_upper(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, double* out,
                         int64_t ldo, int stage, ora_info* info) {
  for (int64_t k = 0; k < n; k++)
    if (T[k * n + k] == 0.0 || !isfinite(T[k * n + k])) return set_err(info, ORA_ESINGULAR, stage, k);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; i++) {
    const double* a = A + i * lda;
    double* o = out + i * ldo;
    for (int64_t k = 0; k < n; k++) {
      double acc = a[k];
      for (int64_t kk = 0; kk < k; kk++) acc -= o[kk] * T[kk * n + k];
      o[k] = acc / T[k * n + k];
    }
  }
  return ORA_OK;
}

/* G = A^T A, upper triangle summed per chunk of <= 64 rows (ascending),
 * chunk partials combined pairwise, then mirrored: exactly symmetric. */
void ora_gram(const double* A, int64_t rows, int64_t n, int64_t lda, double* G) {
  const int64_t CH = 64;
  int64_t nch = (rows + CH - 1) / CH;
  if (nch < 1) nch = 1;
  double* part = (double*)calloc((size_t)(nch * n * n), sizeof(double));
  #pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nch; c++) {
    double* P = part + c * n * n;
    int64_t r1 = (c + 1) * CH < rows ? (c + 1) * CH : rows;
    for (int64_t r = c * CH; r < r1; r++) {
      const double* a = A + r * lda;
      for (int64_t i = 0; i < n; i++) {
        double ai = a[i];
        for (int64_t j = i; j < n; j++) P[i * n + j] += ai * a[j];
      }
    }
  }
  for (int64_t step = 1; step < nch; step *= 2)
    for (int64_t c = 0; c + step < nch; c += 2 * step) {
      double* P = part + c * n * n; const double* Q = part + (c + step) * n * n;
      for (int64_t t = 0; t < n * n; t++) P[t] += Q[t];
    }
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = i; j < n; j++) { G[i * n + j] = part[i * n + j]; G[j * n + i] = part[i * n + j]; }
  free(part);
}

/* R = Cholesky(G), upper, unblocked; a pivot <= 0 or non-finite ->
 * EBREAKDOWN(stage, k). */
int ora_chol(const double* G, int64_t n, double* R, int stage, ora_info* info) {
  memset(R, 0, sizeof(double) * (size_t)(n * n));
  for (int64_t k = 0; k < n; k++) {
    double d = G[k * n + k];
    for (int64_t i = 0; i < k; i++) d -= R[i * n + k] * R[i * n + k];
    if (!(d > 0.0) || !isfinite(d)) return set_err(info, ORA_EBREAKDOWN, stage, k);
    double rkk = sqrt(d);
    R[k * n + k] = rkk;
    for (int64_t j = k + 1; j < n; j++) {
      double a = G[k * n + j];
      for (int64_t i = 0; i < k; i++) a -= R[i * n + k] * R[i * n + j];
      R[k * n + j] = a / rkk;
    }
  }
  return ORA_OK;
}

/* ------------------------------------------------------------ algorithms */
typedef struct {
  double* U; double* L11;   /* n x n (LU) */
  double* Lt;               /* s1 x n CountSketch stage (SSLHC3 only) */
  double* Ls;               /* s x n or s2 x n sketch handed to HouseholderQR */
  double* S; double* Y;     /* n x n */
  double* G1; double* D; double* G2; double* J; /* n x n */
} ora_stages;

static int check_finite(const double* X, int64_t m, int64_t n, int64_t ldx, ora_info* info) {
  for (int64_t i = 0; i < m; i++)
    for (int64_t j = 0; j < n; j++)
      if (!isfinite(X[i * ldx + j])) return set_err(info, ORA_ENONFINITE, ST_INPUT, i * n + j);
  return ORA_OK;
}

/* Shared tail of SLHC3 and SSLHC3 once the sketch L_s /
 * L_ss is known: [H,S] = HouseholderQR(L_s), sign fix (R#7), Y = S U,
 * W = X Y^{-1}, [Q,Z] = CholeskyQR2(W), R = Z Y evaluated
 * as J (D Y) (R#10).  Q (m x n, ldq) holds W, V and Q in turn. */
static int lhc_tail(const double* X, int64_t m, int64_t n, int64_t ldx, double* Ls, int64_t srows,
                    const double* U, double* Q, int64_t ldq, double* R, ora_stages* st, ora_info* info) {
  size_t nn = (size_t)(n * n);
  double* S = (double*)malloc(sizeof(double) * nn);
  double* Y = (double*)malloc(sizeof(double) * nn);
  double* G = (double*)malloc(sizeof(double) * nn);
  double* D = (double*)malloc(sizeof(double) * nn);
  double* J = (double*)malloc(sizeof(double) * nn);
  double* N = (double*)malloc(sizeof(double) * nn);
  double* A = (double*)malloc(sizeof(double) * (size_t)(srows * n));
  memcpy(A, Ls, sizeof(double) * (size_t)(srows * n));
  int rc = ora_hqr_r(A, srows, n, S, info);
  if (rc) goto out;
  for (int64_t k = 0; k < n; k++) /* sign(S_kk) := sign(U_kk) (R#7) */
    if ((S[k * n + k] < 0.0) != (U[k * n + k] < 0.0))
      for (int64_t j = 0; j < n; j++) S[k * n + j] = -S[k * n + j];
  ora_trmm_uu(S, U, n, Y);
  if (st && st->S) memcpy(st->S, S, sizeof(double) * nn);
  if (st && st->Y) memcpy(st->Y, Y, sizeof(double) * nn);
  rc = ora_trsm_right_upper(X, m, n, ldx, Y, Q, ldq, ST_SOLVE_Y, info);          /* W */
  if (rc) goto out;
  ora_gram(Q, m, n, ldq, G);
  if (st && st->G1) memcpy(st->G1, G, sizeof(double) * nn);
  rc = ora_chol(G, n, D, ST_CHOL1, info);
  if (rc) goto out;
  rc = ora_trsm_right_upper(Q, m, n, ldq, D, Q, ldq, ST_SOLVE_D, info);          /* V */
  if (rc) goto out;
  ora_gram(Q, m, n, ldq, G);
  if (st && st->G2) memcpy(st->G2, G, sizeof(double) * nn);
  rc = ora_chol(G, n, J, ST_CHOL2, info);
  if (rc) goto out;
  rc = ora_trsm_right_upper(Q, m, n, ldq, J, Q, ldq, ST_SOLVE_J, info);          /* Q */
  if (rc) goto out;
  ora_trmm_uu(D, Y, n, N);
  ora_trmm_uu(J, N, n, R);
  if (st && st->D) memcpy(st->D, D, sizeof(double) * nn);
  if (st && st->J) memcpy(st->J, J, sizeof(double) * nn);
out:
  free(S); free(Y); free(G); free(D); free(J); free(N); free(A);
  return rc;
}

/* SLHC3 = SLHC + CholeskyQR2.  L_s = Omega L with Omega
 * s x m Gaussian (stream 0), L in original row order (R#2). */
int ora_slhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s, uint64_t seed, int64_t leaf_rows,
              int64_t arity, int64_t panel, double* Q, int64_t ldq, double* R, int64_t* piv, ora_stages* st,
              ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || s < n || s > m || ldx < n || ldq < n) return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  double* U = (double*)malloc(sizeof(double) * nn);
  double* L11 = (double*)malloc(sizeof(double) * nn);
  double* Ls = (double*)malloc(sizeof(double) * (size_t)(s * n));
  double* Lrows = NULL;
  rc = ora_tslu(X, m, n, ldx, leaf_rows, arity, panel, piv, U, L11, NULL, info);
  if (rc) goto out;
  if (st && st->U) memcpy(st->U, U, sizeof(double) * nn);
  if (st && st->L11) memcpy(st->L11, L11, sizeof(double) * nn);
  Lrows = (double*)malloc(sizeof(double) * (size_t)(m * n));
  ora_lfactor(X, m, n, ldx, piv, U, L11, Lrows);
  ora_sketch_gauss(Lrows, m, n, n, 0, s, seed, 0u, Ls);
  free(Lrows); Lrows = NULL;
  if (st && st->Ls) memcpy(st->Ls, Ls, sizeof(double) * (size_t)(s * n));
  rc = lhc_tail(X, m, n, ldx, Ls, s, U, Q, ldq, R, st, info);
out:
  free(U); free(L11); free(Ls); free(Lrows);
  return rc;
}

/* SSLHC3 = SSLHC + CholeskyQR2.  L_t = Omega_1 L
 * (CountSketch, s1 x m), L_ss = Omega_2 L_t (Gaussian s2 x s1, stream 1). */
int ora_sslhc3(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed,
               int64_t leaf_rows, int64_t arity, int64_t panel, double* Q, int64_t ldq, double* R, int64_t* piv,
               ora_stages* st, ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || s2 < n || s1 < s2 || s1 > m || ldx < n || ldq < n)
    return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  double* U = (double*)malloc(sizeof(double) * nn);
  double* L11 = (double*)malloc(sizeof(double) * nn);
  double* Lt = (double*)malloc(sizeof(double) * (size_t)(s1 * n));
  double* Lss = (double*)malloc(sizeof(double) * (size_t)(s2 * n));
  int32_t* bucket = NULL; int8_t* sign = NULL; double* Lrows = NULL;
  rc = ora_tslu(X, m, n, ldx, leaf_rows, arity, panel, piv, U, L11, NULL, info);
  if (rc) goto out;
  if (st && st->U) memcpy(st->U, U, sizeof(double) * nn);
  if (st && st->L11) memcpy(st->L11, L11, sizeof(double) * nn);
  Lrows = (double*)malloc(sizeof(double) * (size_t)(m * n));
  ora_lfactor(X, m, n, ldx, piv, U, L11, Lrows);
  bucket = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  sign = (int8_t*)malloc((size_t)m);
  ora_cs_hash(seed, 0, m, s1, bucket, sign);
  ora_cs_apply(Lrows, m, n, n, bucket, sign, s1, Lt);
  free(Lrows); Lrows = NULL;
  if (st && st->Lt) memcpy(st->Lt, Lt, sizeof(double) * (size_t)(s1 * n));
  ora_sketch_gauss(Lt, s1, n, n, 0, s2, seed, 1u, Lss);
  if (st && st->Ls) memcpy(st->Ls, Lss, sizeof(double) * (size_t)(s2 * n));
  rc = lhc_tail(X, m, n, ldx, Lss, s2, U, Q, ldq, R, st, info);
out:
  free(U); free(L11); free(Lt); free(Lss); free(bucket); free(sign); free(Lrows);
  return rc;
}

/* ------------------------------------------------------------ comparison algorithms */
/* The paper's comparison methods, each step in the paper's order from
 * the primitives above.  Stage tags: the Cholesky of the preconditioning step is ST_CHOL0,
 * the CholeskyQR(2) tail uses ST_CHOL1 / ST_CHOL2 like SLHC3. */

/* CholeskyQR (alg:cholqr) in place on the m x n rows of Q: G = Q^T Q (+ shift I),
 * T = Cholesky(G), Q := Q T^{-1} (substitution). */
static int cholqr_step(double* Q, int64_t m, int64_t n, int64_t ldq, double* T, double shift, int chol_stage,
                       int solve_stage, ora_info* info) {
  double* G = (double*)malloc(sizeof(double) * (size_t)(n * n));
  ora_gram(Q, m, n, ldq, G);
  if (shift != 0.0)
    for (int64_t k = 0; k < n; k++) G[k * n + k] += shift;
  int rc = ora_chol(G, n, T, chol_stage, info);
  if (!rc) rc = ora_trsm_right_upper(Q, m, n, ldq, T, Q, ldq, solve_stage, info);
  free(G);
  return rc;
}

static void copy_rows(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq) {
  for (int64_t i = 0; i < m; i++) memcpy(Q + i * ldq, X + i * ldx, sizeof(double) * (size_t)n);
}

/* CholeskyQR2 (alg:cholqr2): [W, Y] = CholeskyQR(X), [Q, Z] = CholeskyQR(W), R = Z Y. */
int ora_cholqr2(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R,
                ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || ldx < n || ldq < n) return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  double* Y = (double*)malloc(sizeof(double) * nn);
  double* Z = (double*)malloc(sizeof(double) * nn);
  copy_rows(X, m, n, ldx, Q, ldq);
  rc = cholqr_step(Q, m, n, ldq, Y, 0.0, ST_CHOL0, ST_SOLVE_Y, info);
  if (!rc) rc = cholqr_step(Q, m, n, ldq, Z, 0.0, ST_CHOL1, ST_SOLVE_D, info);
  if (!rc) ora_trmm_uu(Z, Y, n, R);
  free(Y); free(Z);
  return rc;
}

/* SCholeskyQR3 (alg:Shifted P:48-59, alg:Shifted3 P:61-71): [W, Y] = SCholeskyQR(X) with
 * s = 11 (m n u + (n + 1) u) ||X||_g^2 (u = 2^-53; ||X||_g = the largest column
 * 2-norm, SPEC S:326 -- here sqrt(max diag(X^T X)), R#21), then
 * [Q, Z] = CholeskyQR2(W) = [W2, D] = CholeskyQR(W), [Q, J] = CholeskyQR(W2), R = J (D Y). */
double ora_scholqr_shift(const double* G, int64_t m, int64_t n) {
  double g = 0.0;
  for (int64_t k = 0; k < n; k++) if (G[k * n + k] > g) g = G[k * n + k];
  const double u = 0x1p-53;
  return 11.0 * ((double)m * (double)n * u + (double)(n + 1) * u) * g;
}

int ora_scholqr3(const double* X, int64_t m, int64_t n, int64_t ldx, double* Q, int64_t ldq, double* R,
                 ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || ldx < n || ldq < n) return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  double* G = (double*)malloc(sizeof(double) * nn);
  double* Y = (double*)malloc(sizeof(double) * nn);
  double* D = (double*)malloc(sizeof(double) * nn);
  double* J = (double*)malloc(sizeof(double) * nn);
  double* N = (double*)malloc(sizeof(double) * nn);
  ora_gram(X, m, n, ldx, G);
  const double shift = ora_scholqr_shift(G, m, n);
  for (int64_t k = 0; k < n; k++) G[k * n + k] += shift;
  rc = ora_chol(G, n, Y, ST_CHOL0, info);
  if (!rc) rc = ora_trsm_right_upper(X, m, n, ldx, Y, Q, ldq, ST_SOLVE_Y, info);
  if (!rc) rc = cholqr_step(Q, m, n, ldq, D, 0.0, ST_CHOL1, ST_SOLVE_D, info);
  if (!rc) rc = cholqr_step(Q, m, n, ldq, J, 0.0, ST_CHOL2, ST_SOLVE_J, info);
  if (!rc) { ora_trmm_uu(D, Y, n, N); ora_trmm_uu(J, N, n, R); }
  free(G); free(Y); free(D); free(J); free(N);
  return rc;
}

/* LUC2 (alg:LU P:75-87, alg:LU2 P:89-99): PX = LU (the tournament contract, R#3), G = L^T L,
 * S = Cholesky(G) ("B" read as G), Y = S U with rows flipped to diag(Y) > 0
 * (R#23: the unique R with a positive diagonal), W = X Y^{-1}; [Q, Z] = CholeskyQR(W), R = Z Y. */
int ora_luc2(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t leaf_rows, int64_t arity, int64_t panel,
             double* Q, int64_t ldq, double* R, int64_t* piv, ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || ldx < n || ldq < n) return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  double* U = (double*)malloc(sizeof(double) * nn);
  double* L11 = (double*)malloc(sizeof(double) * nn);
  double* G = (double*)malloc(sizeof(double) * nn);
  double* S = (double*)malloc(sizeof(double) * nn);
  double* Y = (double*)malloc(sizeof(double) * nn);
  double* Z = (double*)malloc(sizeof(double) * nn);
  double* Lrows = NULL;
  rc = ora_tslu(X, m, n, ldx, leaf_rows, arity, panel, piv, U, L11, NULL, info);
  if (rc) goto out;
  Lrows = (double*)malloc(sizeof(double) * (size_t)(m * n));
  ora_lfactor(X, m, n, ldx, piv, U, L11, Lrows);
  ora_gram(Lrows, m, n, n, G);
  rc = ora_chol(G, n, S, ST_CHOL0, info);
  if (rc) goto out;
  ora_trmm_uu(S, U, n, Y);
  for (int64_t k = 0; k < n; k++) /* diag(Y) > 0 (the sign of U_kk, R#23) */
    if (Y[k * n + k] < 0.0)
      for (int64_t j = 0; j < n; j++) Y[k * n + j] = -Y[k * n + j];
  rc = ora_trsm_right_upper(X, m, n, ldx, Y, Q, ldq, ST_SOLVE_Y, info);
  if (rc) goto out;
  rc = cholqr_step(Q, m, n, ldq, Z, 0.0, ST_CHOL1, ST_SOLVE_D, info);
  if (!rc) ora_trmm_uu(Z, Y, n, R);
out:
  free(U); free(L11); free(G); free(S); free(Y); free(Z); free(Lrows);
  return rc;
}

/* RHC (alg:Rand1 P:103-113, alg:Rand2 P:115-127): K = Omega_2 Omega_1 X (CountSketch s1 x m,
 * stream 2, then Gaussian s2 x s1, stream 1 -- the SSLHC3 sketches applied to X),
 * [H, Y] = HouseholderQR(K) with rows of Y flipped to a positive diagonal (R#22),
 * W = X Y^{-1}; [Q, Z] = CholeskyQR(W), R = Z Y. */
int ora_rhc(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t s1, int64_t s2, uint64_t seed, double* Q,
            int64_t ldq, double* R, ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  if (m < n || n < 1 || s2 < n || s1 < s2 || s1 > m || ldx < n || ldq < n)
    return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  int rc = check_finite(X, m, n, ldx, info);
  if (rc) return rc;
  size_t nn = (size_t)(n * n);
  int32_t* bucket = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  int8_t* sign = (int8_t*)malloc((size_t)m);
  double* Kt = (double*)malloc(sizeof(double) * (size_t)(s1 * n));
  double* K = (double*)malloc(sizeof(double) * (size_t)(s2 * n));
  double* Xc = (double*)malloc(sizeof(double) * (size_t)(m * n));
  double* Y = (double*)malloc(sizeof(double) * nn);
  double* Z = (double*)malloc(sizeof(double) * nn);
  copy_rows(X, m, n, ldx, Xc, n);
  ora_cs_hash(seed, 0, m, s1, bucket, sign);
  ora_cs_apply(Xc, m, n, n, bucket, sign, s1, Kt);
  ora_sketch_gauss(Kt, s1, n, n, 0, s2, seed, 1u, K);
  rc = ora_hqr_r(K, s2, n, Y, info);
  if (rc) goto out;
  for (int64_t k = 0; k < n; k++)
    if (Y[k * n + k] < 0.0)
      for (int64_t j = 0; j < n; j++) Y[k * n + j] = -Y[k * n + j];
  rc = ora_trsm_right_upper(X, m, n, ldx, Y, Q, ldq, ST_SOLVE_Y, info);
  if (rc) goto out;
  rc = cholqr_step(Q, m, n, ldq, Z, 0.0, ST_CHOL1, ST_SOLVE_D, info);
  if (!rc) ora_trmm_uu(Z, Y, n, R);
out:
  free(bucket); free(sign); free(Kt); free(K); free(Xc); free(Y); free(Z);
  return rc;
}

/* ------------------------------------------------------------ checkers */
/* Orthogonality ||Q^T Q - I||_F and relative residual ||QR - X||_F / ||X||_F
 * with long-double accumulation (R#16, exp5). */
double ora_orthogonality(const double* Q, int64_t m, int64_t n, int64_t ldq) {
  long double tot = 0.0L;
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = i; j < n; j++) {
      long double g = 0.0L;
      for (int64_t r = 0; r < m; r++) g += (long double)Q[r * ldq + i] * (long double)Q[r * ldq + j];
      if (i == j) g -= 1.0L;
      tot += (i == j ? 1.0L : 2.0L) * g * g;
    }
  return (double)sqrtl(tot);
}

double ora_residual(const double* Q, const double* R, const double* X, int64_t m, int64_t n, int64_t ldq,
                    int64_t ldx) {
  long double num = 0.0L, den = 0.0L;
  for (int64_t r = 0; r < m; r++)
    for (int64_t j = 0; j < n; j++) {
      long double acc = 0.0L;
      for (int64_t k = 0; k <= j; k++) acc += (long double)Q[r * ldq + k] * (long double)R[k * n + j];
      long double x = X[r * ldx + j];
      num += (acc - x) * (acc - x);
      den += x * x;
    }
  return (double)sqrtl(num / den);
}

/* ---------------------------------------------- pieces for the row-sharded check */
/* (Used only by tests/test_dist_cpu.py: the oracle-side stages of one rank.  Same
 * arithmetic as ora_tslu, split at the points where the distributed algorithm exchanges
 * data.) */

/* GEPP selection on cnt candidate rows (B, cnt x w, overwritten), R#4-R#5 */
int64_t ora_select(double* B, const int64_t* ids, int64_t cnt, int64_t w, int64_t* out_ids) {
  return gepp_select(B, ids, cnt, w, out_ids);
}

/* U rows of one panel from its w pivot rows (prow, w x ncols, pivot order, columns
 * p0..p0+ncols-1): the elimination of ora_tslu restricted to the pivot rows. */
void ora_panel_rows(double* prow, int64_t w, int64_t ncols) {
  for (int64_t k = 0; k < w; k++) {
    double r = 1.0 / prow[k * ncols + k];
    for (int64_t t = k + 1; t < w; t++) {
      double l = prow[t * ncols + k] * r;
      prow[t * ncols + k] = l;
      for (int64_t j = k + 1; j < ncols; j++) prow[t * ncols + j] = fma(-l, prow[k * ncols + j], prow[t * ncols + j]);
    }
  }
}

/* eliminate rows (A, rows x n, current values) with the panel pivots k = p0..p0+w-1 of U
 * (skipping rows flagged in chosen): the elimination loop of ora_tslu. */
void ora_eliminate_rows(double* A, int64_t rows, int64_t n, int64_t p0, int64_t w, const double* U,
                        const unsigned char* chosen) {
  for (int64_t k = p0; k < p0 + w; k++) {
    double r = 1.0 / U[k * n + k];
    for (int64_t i = 0; i < rows; i++) {
      if (chosen && chosen[i]) continue;
      double* a = A + i * n;
      double l = a[k] * r;
      a[k] = l;
      for (int64_t j = k + 1; j < n; j++) a[j] = fma(-l, U[k * n + j], a[j]);
    }
  }
}

/* L rows of X rows with global ids row0.. (pivot rows take L11 rows) */
void ora_lfactor_rows(const double* X, int64_t rows, int64_t n, int64_t row0, const int64_t* piv, const double* U,
                      const double* L11, double* L) {
  double* rd = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t k = 0; k < n; k++) rd[k] = 1.0 / U[k * n + k];
  for (int64_t i = 0; i < rows; i++) {
    int64_t pp = -1;
    for (int64_t k = 0; k < n; k++) if (piv[k] == row0 + i) pp = k;
    l_row(X + i * n, n, U, rd, L11, pp, L + i * n);
  }
  free(rd);
}

/* ------------------------------------------------ row-chunked SLHC3 / SSLHC3 (cfg5) */
/* The same algorithm, step for step and bit for bit, as ora_slhc3 / ora_sslhc3 above, for
 * X too large to hold twice in host RAM (cfg5: 2^24 x 256 = 32 GiB; SURVEY 8(c) "processes X
 * in row chunks").  X is never stored: get(user, row0, rows, buf) delivers rows
 * [row0, row0 + rows) (rows x n, row-major) whenever a pass needs them, and put (optional)
 * receives the rows of Q.  Host memory is O(chunk_rows * n + n^2 + s1 * n + tree), where the
 * tree holds at most arity pending nodes of w winners per level.
 *
 * Every value is the one the in-memory oracle computes:
 *  - TSLU (R#3-R#5): per panel, the leaves' candidate values are the rows'
 *    Schur complements at the panel start, recomputed from the X row by the elimination's own
 *    per-element fma chain (l = a_k * (1/U_kk), a_j = fma(-l, U_kj, a_j), k increasing) --
 *    the right-looking update of ora_tslu applies exactly this sequence to every element.
 *    Nodes are formed as leaves stream in (arity consecutive children; the trailing partial
 *    group of a level closes when the stream ends), so the tree is ora_tslu's tree.  Pivot
 *    row k's U / L11 row is its X row run through pivots 0..k-1 by the same chain.
 *  - L rows by l_row (ora_lfactor), CountSketch in ascending rows (ora_cs_apply), the
 *    Gaussian sketch with ora_sketch_gauss's fixed 64-way row partition.
 *  - W = X Y^-1, V = W D^-1, Q = V J^-1 recomputed per chunk by ora_trsm_right_upper (row
 *    independent); the Grams with ora_gram's 64-row partials combined by its pairwise tree
 *    (a binary-counter stack: merging equal-size neighbours left + right, folding the rest
 *    from the right at the end reproduces ora_gram's step-doubling sums exactly).
 * chunk_rows must be a positive multiple of leaf_rows and of 64. */
typedef void (*ora_rows_fn)(void* user, int64_t row0, int64_t rows, double* buf);
typedef void (*ora_qrows_fn)(void* user, int64_t row0, int64_t rows, const double* Q);

typedef struct { int64_t cnt; int64_t ids[64]; double* vals; } ck_node; /* winners + panel-start values */

typedef struct {
  int64_t w, arity, nlev;
  ck_node* pend;       /* [lev * arity + i] */
  int64_t* npend;      /* pending children per level */
  int64_t* total;      /* nodes ever pushed per level */
  ck_node root;
  int have_root;
} ck_tree;

static void ck_node_free(ck_node* nd) { free(nd->vals); nd->vals = NULL; nd->cnt = 0; }

/* GEPP over the stacked children (their order = global order), winners keep their values */
static ck_node ck_combine(const ck_node* ch, int64_t nch, int64_t w) {
  int64_t tot = 0;
  for (int64_t c = 0; c < nch; c++) tot += ch[c].cnt;
  ck_node out; out.cnt = 0; out.vals = (double*)malloc(sizeof(double) * (size_t)(w * w > 0 ? w * w : 1));
  int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(tot > 0 ? tot : 1));
  double* V = (double*)malloc(sizeof(double) * (size_t)((tot > 0 ? tot : 1) * w));
  double* B = (double*)malloc(sizeof(double) * (size_t)((tot > 0 ? tot : 1) * w));
  int64_t q = 0;
  for (int64_t c = 0; c < nch; c++)
    for (int64_t e = 0; e < ch[c].cnt; e++, q++) {
      ids[q] = ch[c].ids[e];
      memcpy(V + q * w, ch[c].vals + e * w, sizeof(double) * (size_t)w);
    }
  memcpy(B, V, sizeof(double) * (size_t)(tot * w));
  out.cnt = gepp_select(B, ids, tot, w, out.ids);
  for (int64_t t = 0; t < out.cnt; t++) {
    int64_t pos = 0;
    while (ids[pos] != out.ids[t]) pos++;
    memcpy(out.vals + t * w, V + pos * w, sizeof(double) * (size_t)w);
  }
  free(ids); free(V); free(B);
  return out;
}

static void ck_push(ck_tree* T, int64_t lev, ck_node nd) {
  if (lev >= T->nlev) { /* grow */
    int64_t nl = T->nlev * 2 + 4;
    T->pend = (ck_node*)realloc(T->pend, sizeof(ck_node) * (size_t)(nl * T->arity));
    T->npend = (int64_t*)realloc(T->npend, sizeof(int64_t) * (size_t)nl);
    T->total = (int64_t*)realloc(T->total, sizeof(int64_t) * (size_t)nl);
    for (int64_t l = T->nlev; l < nl; l++) { T->npend[l] = 0; T->total[l] = 0; }
    T->nlev = nl;
  }
  T->pend[lev * T->arity + T->npend[lev]++] = nd;
  T->total[lev]++;
  if (T->npend[lev] == T->arity) {
    ck_node parent = ck_combine(T->pend + lev * T->arity, T->arity, T->w);
    for (int64_t i = 0; i < T->arity; i++) ck_node_free(T->pend + lev * T->arity + i);
    T->npend[lev] = 0;
    ck_push(T, lev + 1, parent);
  }
}

/* end of the stream: close every level's trailing partial group, bottom up */
static void ck_finish(ck_tree* T) {
  for (int64_t lev = 0; lev < T->nlev; lev++) {
    if (T->total[lev] == 1 && T->npend[lev] == 1) { /* the only node of its level: the root */
      T->root = T->pend[lev * T->arity];
      T->npend[lev] = 0;
      T->have_root = 1;
      return;
    }
    if (T->npend[lev] > 0) {
      ck_node parent = ck_combine(T->pend + lev * T->arity, T->npend[lev], T->w);
      for (int64_t i = 0; i < T->npend[lev]; i++) ck_node_free(T->pend + lev * T->arity + i);
      T->npend[lev] = 0;
      ck_push(T, lev + 1, parent);
    }
  }
}

/* a row's current values after pivots 0..K-1 (columns < jmax): the elimination chain */
static void ck_eliminate(double* a, int64_t K, int64_t jmax, int64_t n, const double* U, const double* rd) {
  for (int64_t k = 0; k < K; k++) {
    double l = a[k] * rd[k];
    a[k] = l;
    for (int64_t j = k + 1; j < jmax; j++) a[j] = fma(-l, U[k * n + j], a[j]);
  }
}

/* row of L (l_row's values): a pivot row takes its L11 row, any other row is its X row run
 * through all n pivots by the elimination chain -- per element the same fma sequence as
 * l_row's substitution (k increasing), evaluated column-oriented so it vectorises */
static void ck_lrow(const double* x, int64_t n, const double* U, const double* rd, const double* L11, int64_t pp,
                    double* l) {
  if (pp >= 0) { memcpy(l, L11 + pp * n, sizeof(double) * (size_t)n); return; }
  memcpy(l, x, sizeof(double) * (size_t)n);
  ck_eliminate(l, n, n, n, U, rd);
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}

/* position k of row id in piv[0..cnt) (sorted copy with positions), -1 if not a pivot */
typedef struct { int64_t id, k; } ck_pp;
static int cmp_pp(const void* a, const void* b) {
  int64_t x = ((const ck_pp*)a)->id, y = ((const ck_pp*)b)->id;
  return x < y ? -1 : x > y;
}
static int64_t ck_pivpos(const ck_pp* srt, int64_t cnt, int64_t id) {
  int64_t lo = 0, hi = cnt;
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (srt[mid].id < id) lo = mid + 1; else hi = mid; }
  return (lo < cnt && srt[lo].id == id) ? srt[lo].k : -1;
}

/* out = A T^{-1}: ora_trsm_right_upper's per-element sequence (acc = a_k; acc -= o_j T_jk as a
 * rounded product then a rounded difference, j increasing; o_k = acc / T_kk) evaluated
 * column-oriented (o_k final before it is used), so the loop over later columns is
 * independent per element and vectorises; every element sees the identical operation
 * sequence (tests/test_oracle_chunked.py checks the bits against ora_trsm_right_upper). */
static int ck_trsm(const double* A, int64_t rows, int64_t n, const double* T, double* out, int stage,
                   ora_info* info) {
  for (int64_t k = 0; k < n; k++)
    if (T[k * n + k] == 0.0 || !isfinite(T[k * n + k])) return set_err(info, ORA_ESINGULAR, stage, k);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; i++) {
    double* o = out + i * n;
    if (o != A + i * n) memcpy(o, A + i * n, sizeof(double) * (size_t)n);
    for (int64_t k = 0; k < n; k++) {
      double ok = o[k] / T[k * n + k];
      o[k] = ok;
      const double* t = T + k * n;
      for (int64_t j = k + 1; j < n; j++) o[j] -= ok * t[j];
    }
  }
  return ORA_OK;
}

int ora_num_threads(void);

/* Gram partial stack (ora_gram's pairwise tree, streamed).  Buffers are recycled through a
 * free list (a fresh calloc per 64-row partial page-faults 512 KB at n = 256). */
typedef struct { double* P; int64_t size; } ck_gp;
typedef struct { ck_gp* s; int64_t top, cap, nn; double** pool; int64_t npool, cappool; } ck_gstack;
static double* ck_gtake(ck_gstack* g) {
  if (g->npool > 0) return g->pool[--g->npool];
  return (double*)malloc(sizeof(double) * (size_t)g->nn);
}
static void ck_ggive(ck_gstack* g, double* P) {
  if (g->npool == g->cappool) {
    g->cappool = g->cappool * 2 + 8;
    g->pool = (double**)realloc(g->pool, sizeof(double*) * (size_t)g->cappool);
  }
  g->pool[g->npool++] = P;
}
/* push the next 64-row partial (copied): merge equal-size neighbours, left += right */
static void ck_gpush(ck_gstack* g, const double* src) {
  double* cur = ck_gtake(g);
  memcpy(cur, src, sizeof(double) * (size_t)g->nn);
  int64_t size = 1;
  while (g->top > 0 && g->s[g->top - 1].size == size) {
    double* left = g->s[--g->top].P;
    for (int64_t t = 0; t < g->nn; t++) left[t] += cur[t];
    ck_ggive(g, cur);
    cur = left; size *= 2;
  }
  if (g->top == g->cap) { g->cap = g->cap * 2 + 8; g->s = (ck_gp*)realloc(g->s, sizeof(ck_gp) * (size_t)g->cap); }
  g->s[g->top].P = cur; g->s[g->top].size = size; g->top++;
}
static void ck_gfree(ck_gstack* g) {
  while (g->top > 0) free(g->s[--g->top].P);
  while (g->npool > 0) free(g->pool[--g->npool]);
  free(g->s); free(g->pool);
  g->s = NULL; g->pool = NULL; g->cap = g->cappool = 0;
}
static void ck_gfinish(ck_gstack* g, int64_t n, double* G) {
  double* P;
  if (g->top == 0) { P = ck_gtake(g); memset(P, 0, sizeof(double) * (size_t)g->nn); }
  else {
    P = g->s[--g->top].P;
    while (g->top > 0) {
      double* left = g->s[--g->top].P;
      for (int64_t t = 0; t < g->nn; t++) left[t] += P[t];
      ck_ggive(g, P);
      P = left;
    }
  }
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = i; j < n; j++) { G[i * n + j] = P[i * n + j]; G[j * n + i] = P[i * n + j]; }
  ck_ggive(g, P);
  ck_gfree(g);
}
/* 64-row partials of rows (chunks are multiples of 64 rows; only the last may be ragged),
 * computed NT at a time in per-thread buffers, then pushed in row order */
static void ck_gram_rows(ck_gstack* g, const double* A, int64_t rows, int64_t n) {
  const int64_t CH = 64;
  int64_t nch = (rows + CH - 1) / CH;
  int nt = ora_num_threads();
  double* buf = (double*)malloc(sizeof(double) * (size_t)nt * (size_t)(n * n));
  for (int64_t c0 = 0; c0 < nch; c0 += nt) {
    int64_t c1 = c0 + nt < nch ? c0 + nt : nch;
    #pragma omp parallel for schedule(static, 1)
    for (int64_t c = c0; c < c1; c++) {
      double* P = buf + (size_t)(c - c0) * (size_t)(n * n);
      memset(P, 0, sizeof(double) * (size_t)(n * n));
      int64_t r1 = (c + 1) * CH < rows ? (c + 1) * CH : rows;
      /* ora_gram's P[i,j] += a_r[i] a_r[j] over r ascending, tiled over (i, j) so a tile of
       * P stays in L1 (per element the same sequence) */
      for (int64_t ib = 0; ib < n; ib += 32)
        for (int64_t jb = ib; jb < n; jb += 32) {
          int64_t ie = ib + 32 < n ? ib + 32 : n, je = jb + 32 < n ? jb + 32 : n;
          for (int64_t r = c * CH; r < r1; r++) {
            const double* a = A + r * n;
            for (int64_t i = ib; i < ie; i++) {
              double ai = a[i];
              for (int64_t j = (i > jb ? i : jb); j < je; j++) P[i * n + j] += ai * a[j];
            }
          }
        }
    }
    for (int64_t c = c0; c < c1; c++) ck_gpush(g, buf + (size_t)(c - c0) * (size_t)(n * n));
  }
  free(buf);
}

int ora_lhc3_chunked(int algo, int64_t m, int64_t n, int64_t s_or_s1, int64_t s2, uint64_t seed, int64_t b,
                     int64_t arity, int64_t panel, int64_t chunk_rows, ora_rows_fn get, ora_qrows_fn put, void* user,
                     double* R, int64_t* piv, ora_stages* st, ora_info* info) {
  if (info) { info->code = 0; info->stage = 0; info->index = 0; }
  const int sslhc = algo == 1;
  const int64_t s = s_or_s1, s1 = s_or_s1;
  if (m < n || n < 1 || b < 1 || arity < 2 || panel < 1 || panel > 64 || !get || chunk_rows < 1 ||
      chunk_rows % b || chunk_rows % 64)
    return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  if (sslhc ? (s2 < n || s1 < s2 || s1 > m) : (s < n || s > m)) return set_err(info, ORA_EINVAL, ST_INPUT, 0);
  const size_t nn = (size_t)(n * n);
  double* Xc = (double*)malloc(sizeof(double) * (size_t)(chunk_rows * n));
  double* Wc = (double*)malloc(sizeof(double) * (size_t)(chunk_rows * n));
  double* Sv = (double*)malloc(sizeof(double) * (size_t)(chunk_rows * (panel < n ? panel : n)));
  double* U = (double*)calloc(nn, sizeof(double));
  double* L11 = (double*)calloc(nn, sizeof(double));
  double* rd = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* chosen = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t nchosen = 0;
  int rc = ORA_OK;
  /* O0: finite input */
  for (int64_t c0 = 0; c0 < m && rc == ORA_OK; c0 += chunk_rows) {
    int64_t rows = (m - c0) < chunk_rows ? (m - c0) : chunk_rows;
    get(user, c0, rows, Xc);
    for (int64_t t = 0; t < rows * n; t++)
      if (!isfinite(Xc[t])) { rc = set_err(info, ORA_ENONFINITE, ST_INPUT, c0 * n + t); break; }
  }
  /* TSLU over panels */
  for (int64_t p0 = 0; p0 < n && rc == ORA_OK; p0 += panel) {
    const int64_t w = (n - p0) < panel ? (n - p0) : panel;
    ck_tree T = {w, arity, 0, NULL, NULL, NULL, {0, {0}, NULL}, 0};
    for (int64_t c0 = 0; c0 < m; c0 += chunk_rows) {
      int64_t rows = (m - c0) < chunk_rows ? (m - c0) : chunk_rows;
      get(user, c0, rows, Xc);
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < rows; i++) {
        double* a = Xc + i * n;
        ck_eliminate(a, p0, p0 + w, n, U, rd);
        memcpy(Sv + i * w, a + p0, sizeof(double) * (size_t)w);
      }
      int64_t nl = (rows + b - 1) / b;
      ck_node* leaves = (ck_node*)malloc(sizeof(ck_node) * (size_t)nl);
      #pragma omp parallel for schedule(dynamic, 4)
      for (int64_t l = 0; l < nl; l++) {
        int64_t r0 = l * b, r1 = (r0 + b < rows) ? r0 + b : rows;
        ck_node leaf; leaf.cnt = 0;
        leaf.vals = (double*)malloc(sizeof(double) * (size_t)(w * w));
        int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(r1 - r0));
        double* B = (double*)malloc(sizeof(double) * (size_t)((r1 - r0) * w));
        int64_t c = 0;
        for (int64_t i = r0; i < r1; i++) {
          int64_t id = c0 + i;
          if (bsearch(&id, chosen, (size_t)nchosen, sizeof(int64_t), cmp_i64)) continue;
          ids[c] = id;
          memcpy(B + c * w, Sv + i * w, sizeof(double) * (size_t)w);
          c++;
        }
        leaf.cnt = gepp_select(B, ids, c, w, leaf.ids);
        for (int64_t t = 0; t < leaf.cnt; t++) {
          int64_t pos = 0;
          while (ids[pos] != leaf.ids[t]) pos++;
          memcpy(leaf.vals + t * w, Sv + (ids[pos] - c0) * w, sizeof(double) * (size_t)w);
        }
        free(ids); free(B);
        leaves[l] = leaf;
      }
      for (int64_t l = 0; l < nl; l++) ck_push(&T, 0, leaves[l]);
      free(leaves);
    }
    ck_finish(&T);
    if (T.root.cnt < w) rc = set_err(info, ORA_ERANKDEF, ST_LU, p0 + T.root.cnt);
    for (int64_t t = 0; t < w && rc == ORA_OK; t++) piv[p0 + t] = T.root.ids[t];
    ck_node_free(&T.root);
    free(T.pend); free(T.npend); free(T.total);
    /* this panel's U / L11 rows: pivot row k through pivots 0..k-1 */
    for (int64_t k = p0; k < p0 + w && rc == ORA_OK; k++) {
      double* a = Wc;
      get(user, piv[k], 1, a);
      ck_eliminate(a, k, n, n, U, rd);
      if (a[k] == 0.0) { rc = set_err(info, ORA_ERANKDEF, ST_LU, k); break; }
      for (int64_t j = k; j < n; j++) U[k * n + j] = a[j];
      for (int64_t j = 0; j < k; j++) L11[k * n + j] = a[j];
      L11[k * n + k] = 1.0;
      rd[k] = 1.0 / U[k * n + k];
    }
    for (int64_t t = 0; t < w && rc == ORA_OK; t++) chosen[nchosen++] = piv[p0 + t];
    qsort(chosen, (size_t)nchosen, sizeof(int64_t), cmp_i64);
  }
  double *Lt = NULL, *Ls = NULL, *part = NULL;
  double *S = NULL, *Y = NULL, *G = NULL, *D = NULL, *J = NULL, *N = NULL, *A = NULL;
  ck_pp* srt = NULL;
  const int64_t srows = sslhc ? s2 : s;
  if (rc) goto out;
  if (st && st->U) memcpy(st->U, U, sizeof(double) * nn);
  if (st && st->L11) memcpy(st->L11, L11, sizeof(double) * nn);
  for (int64_t k = 0; k < n; k++) rd[k] = 1.0 / U[k * n + k];
  srt = (ck_pp*)malloc(sizeof(ck_pp) * (size_t)n);
  for (int64_t k = 0; k < n; k++) { srt[k].id = piv[k]; srt[k].k = k; }
  qsort(srt, (size_t)n, sizeof(ck_pp), cmp_pp);
  /* L rows and their sketch (P:280 / P:294) */
  Ls = (double*)malloc(sizeof(double) * (size_t)(srows * n));
  if (sslhc) {
    Lt = (double*)calloc((size_t)(s1 * n), sizeof(double));
    int32_t* bucket = (int32_t*)malloc(sizeof(int32_t) * (size_t)chunk_rows);
    int8_t* sign = (int8_t*)malloc((size_t)chunk_rows);
    for (int64_t c0 = 0; c0 < m; c0 += chunk_rows) {
      int64_t rows = (m - c0) < chunk_rows ? (m - c0) : chunk_rows;
      get(user, c0, rows, Xc);
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < rows; i++) ck_lrow(Xc + i * n, n, U, rd, L11, ck_pivpos(srt, n, c0 + i), Wc + i * n);
      ora_cs_hash(seed, c0, rows, s1, bucket, sign);
      for (int64_t j = 0; j < rows; j++) { /* ora_cs_apply's ascending-row accumulation */
        double* o = Lt + (int64_t)bucket[j] * n;
        const double* a = Wc + j * n;
        if (sign[j] > 0) for (int64_t c = 0; c < n; c++) o[c] += a[c];
        else             for (int64_t c = 0; c < n; c++) o[c] -= a[c];
      }
    }
    free(bucket); free(sign);
    if (st && st->Lt) memcpy(st->Lt, Lt, sizeof(double) * (size_t)(s1 * n));
    ora_sketch_gauss(Lt, s1, n, n, 0, s2, seed, 1u, Ls);
  } else {
    /* ora_sketch_gauss's 64 partials over the fixed row partition [m ch/64, m (ch+1)/64) */
    const int NCH = 64;
    part = (double*)calloc((size_t)NCH * s * n, sizeof(double));
    for (int64_t c0 = 0; c0 < m; c0 += chunk_rows) {
      int64_t rows = (m - c0) < chunk_rows ? (m - c0) : chunk_rows;
      get(user, c0, rows, Xc);
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < rows; i++) ck_lrow(Xc + i * n, n, U, rd, L11, ck_pivpos(srt, n, c0 + i), Wc + i * n);
      #pragma omp parallel for schedule(static)
      for (int ch = 0; ch < NCH; ch++) {
        int64_t a0 = m * ch / NCH, a1 = m * (ch + 1) / NCH;
        if (a0 < c0) a0 = c0;
        if (a1 > c0 + rows) a1 = c0 + rows;
        double* P = part + (size_t)ch * s * n;
        double* om = (double*)malloc(sizeof(double) * (size_t)s);
        for (int64_t j = a0; j < a1; j++) {
          for (int64_t i = 0; i < s; i += 2) {
            double z0, z1;
            ora_gauss_pair(seed, (uint64_t)j, (uint32_t)(i >> 1), 0u, &z0, &z1);
            double sc = 1.0 / sqrt((double)s);
            om[i] = z0 * sc;
            if (i + 1 < s) om[i + 1] = z1 * sc;
          }
          const double* a = Wc + (j - c0) * n;
          for (int64_t i = 0; i < s; i++) {
            double wv = om[i];
            double* p = P + i * n;
            for (int64_t c = 0; c < n; c++) p[c] += wv * a[c];
          }
        }
        free(om);
      }
    }
    memset(Ls, 0, sizeof(double) * (size_t)(s * n));
    for (int ch = 0; ch < NCH; ch++)
      for (int64_t t = 0; t < s * n; t++) Ls[t] += part[(size_t)ch * s * n + t];
  }
  if (st && st->Ls) memcpy(st->Ls, Ls, sizeof(double) * (size_t)(srows * n));
  /* the tail of lhc_tail, with W and V recomputed per chunk */
  S = (double*)malloc(sizeof(double) * nn); Y = (double*)malloc(sizeof(double) * nn);
  G = (double*)malloc(sizeof(double) * nn); D = (double*)malloc(sizeof(double) * nn);
  J = (double*)malloc(sizeof(double) * nn); N = (double*)malloc(sizeof(double) * nn);
  A = (double*)malloc(sizeof(double) * (size_t)(srows * n));
  memcpy(A, Ls, sizeof(double) * (size_t)(srows * n));
  rc = ora_hqr_r(A, srows, n, S, info);
  if (rc) goto out;
  for (int64_t k = 0; k < n; k++)
    if ((S[k * n + k] < 0.0) != (U[k * n + k] < 0.0))
      for (int64_t j = 0; j < n; j++) S[k * n + j] = -S[k * n + j];
  ora_trmm_uu(S, U, n, Y);
  if (st && st->S) memcpy(st->S, S, sizeof(double) * nn);
  if (st && st->Y) memcpy(st->Y, Y, sizeof(double) * nn);
  for (int pass = 0; pass < 3 && rc == ORA_OK; pass++) {
    ck_gstack gs = {NULL, 0, 0, (int64_t)nn, NULL, 0, 0};
    for (int64_t c0 = 0; c0 < m && rc == ORA_OK; c0 += chunk_rows) {
      int64_t rows = (m - c0) < chunk_rows ? (m - c0) : chunk_rows;
      get(user, c0, rows, Xc);
      rc = ck_trsm(Xc, rows, n, Y, Wc, ST_SOLVE_Y, info);                 /* W */
      if (!rc && pass >= 1) rc = ck_trsm(Wc, rows, n, D, Wc, ST_SOLVE_D, info); /* V */
      if (!rc && pass >= 2) rc = ck_trsm(Wc, rows, n, J, Wc, ST_SOLVE_J, info); /* Q */
      if (rc) break;
      if (pass < 2) ck_gram_rows(&gs, Wc, rows, n);
      else if (put) put(user, c0, rows, Wc);
    }
    if (rc) { ck_gfree(&gs); break; }
    if (pass == 0) {
      ck_gfinish(&gs, n, G);
      if (st && st->G1) memcpy(st->G1, G, sizeof(double) * nn);
      rc = ora_chol(G, n, D, ST_CHOL1, info);
    } else if (pass == 1) {
      ck_gfinish(&gs, n, G);
      if (st && st->G2) memcpy(st->G2, G, sizeof(double) * nn);
      rc = ora_chol(G, n, J, ST_CHOL2, info);
    } else {
      ck_gfree(&gs);
    }
  }
  if (rc) goto out;
  ora_trmm_uu(D, Y, n, N);
  ora_trmm_uu(J, N, n, R);
  if (st && st->D) memcpy(st->D, D, sizeof(double) * nn);
  if (st && st->J) memcpy(st->J, J, sizeof(double) * nn);
out:
  free(Xc); free(Wc); free(Sv); free(U); free(L11); free(rd); free(chosen); free(srt);
  free(Lt); free(Ls); free(part); free(S); free(Y); free(G); free(D); free(J); free(N); free(A);
  return rc;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
