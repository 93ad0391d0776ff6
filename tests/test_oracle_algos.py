"""Pins for the oracle's end-to-end SLHC3 / SSLHC3.  In exact arithmetic
the output (Q, R with diag R > 0) is the unique thin QR of X, independent of the
sketch, the seed and the pivots -- so it is pinned against LAPACK, a long-double
Gram-Schmidt, mpmath, and the theorems' bounds and the paper's own
experiment magnitudes."""
import math

import numpy as np
import pytest

import synth
from conftest import orth_err, qr_signed, rel_fro, rel_residual

U_ROUND = 2.0 ** -53


def _x(m, n, kexp, seed, colscale=False):
    return synth.baseline_matrix(m, n, kexp, seed, colscale).numpy()


def _run(ora, algo, X, seed=0, s=None, s1=None, s2=None, b=None, a=4, panel=None, **kw):
    m, n = X.shape
    b = b or max(2 * n, 64)
    if algo == "slhc3":
        return ora.slhc3(X, s or 2 * n, seed, b, a, panel, **kw)
    return ora.sslhc3(X, s1 or min(8 * n, m), s2 or 2 * n, seed, b, a, panel, **kw)


@pytest.mark.parametrize("algo", ["slhc3", "sslhc3"])
def test_identity(ora, algo):
    """X = I_n -> Q = I, R = I.  SSLHC3 needs a CountSketch that
    embeds range(L), so its identity is padded with zero rows: X = [I; 0]
    with s1 = m (a square X = I_n hashed into n buckets collides and is not an embedding)."""
    n = 4
    if algo == "slhc3":
        X = np.eye(n)
        r = ora.slhc3(X, n, 0, 8, 2)
    else:
        X = np.zeros((1024, n)); X[:n] = np.eye(n)
        r = ora.sslhc3(X, 1024, n, 0, 64, 2)
    assert np.allclose(r.Q, X, atol=1e-15) and np.allclose(r.R, np.eye(n), atol=1e-15)


@pytest.mark.parametrize("algo,m,n,kexp,colscale", [
    ("slhc3", 2048, 16, 8, False),     # cfg1
    ("slhc3", 8192, 48, 12, False),
    ("sslhc3", 16384, 32, 15, True),   # cfg3-like (column scaling)
    ("sslhc3", 4096, 64, 10, False),
])
def test_gates_and_unique_qr(ora, algo, m, n, kexp, colscale):
    """BASELINE gates (orthogonality <= 1e-13 sqrt(n), residual <= 1e-14 n) and R against
    the unique sign-normalised LAPACK QR.  diag(R) > 0 holds by construction (R#7)."""
    X = _x(m, n, kexp, 3, colscale)
    r = _run(ora, algo, X, seed=5)
    assert np.all(np.diag(r.R) > 0)
    assert np.array_equal(np.tril(r.R, -1), np.zeros((n, n)))
    assert orth_err(r.Q) <= 1e-13 * math.sqrt(n)
    assert rel_residual(r.Q, r.R, X) <= 1e-14 * n
    Ql, Rl = qr_signed(X)
    if kexp <= 8 and not colscale:
        assert rel_fro(r.R, Rl) <= 1e-12       # BJ: <= 1e-9 for kappa <= 1e8
    # theorem 3.3 / 3.4 orthogonality bound
    assert orth_err(r.Q) <= 6 * (m * n * U_ROUND + n * (n + 1) * U_ROUND)


def test_seed_and_pivot_invariance_of_R(ora):
    """R is the unique thin-QR factor: independent of the sketch seed and of the
    tournament shape (leaf size / arity / panel) up to rounding (exp6: 2-4e-16)."""
    X = _x(4096, 24, 8, 1)
    R0 = _run(ora, "slhc3", X, seed=1).R
    for kw in [dict(seed=2), dict(seed=3, b=512, a=2), dict(seed=4, panel=8), dict(seed=5, b=4096)]:
        assert rel_fro(_run(ora, "slhc3", X, **kw).R, R0) < 1e-13
    assert rel_fro(_run(ora, "sslhc3", X, seed=7).R, R0) < 1e-13


def test_long_double_gram_schmidt(ora):
    """Brute force: R from CGS2 in extended precision (np.longdouble) on a small input."""
    X = _x(400, 10, 6, 2)
    Xl = X.astype(np.longdouble)
    m, n = X.shape
    Q = np.zeros((m, n), np.longdouble); R = np.zeros((n, n), np.longdouble)
    for j in range(n):
        v = Xl[:, j].copy()
        for _ in range(2):
            c = Q[:, :j].T @ v
            v -= Q[:, :j] @ c
            R[:j, j] += c
        R[j, j] = np.sqrt(v @ v)
        Q[:, j] = v / R[j, j]
    r = _run(ora, "slhc3", X, seed=3)
    assert rel_fro(r.R, R.astype(np.float64)) < 1e-13
    assert rel_fro(r.Q, Q.astype(np.float64)) < 1e-9


def test_mpmath_tiny(ora):
    import mpmath
    mpmath.mp.dps = 40
    X = _x(40, 5, 4, 6)
    A = mpmath.matrix(X.tolist())
    Q, R = mpmath.qr(A)
    Rm = np.array([[float(R[i, j]) for j in range(5)] for i in range(5)])
    d = np.sign(np.diag(Rm)); Rm = Rm * d[:, None]
    for algo in ("slhc3", "sslhc3"):
        r = _run(ora, algo, X, s1=20, s2=10, s=10, b=16)
        assert rel_fro(r.R, Rm) < 1e-14


def test_equivariances(ora):
    """X D -> R D (column scaling by powers of 2 is exact); Pi X -> (Pi Q, R)."""
    X = _x(2048, 16, 8, 4)
    r = _run(ora, "slhc3", X, seed=2)
    D = 2.0 ** np.arange(-8, 8)
    rd = _run(ora, "slhc3", X * D, seed=2)
    assert rel_fro(rd.R, r.R * D) < 1e-13
    perm = np.random.default_rng(0).permutation(2048)
    rp = _run(ora, "slhc3", X[perm], seed=2)
    assert rel_fro(rp.R, r.R) < 1e-13
    # Q is determined only to ~ kappa * u (here kappa = 1e8)
    assert np.linalg.norm(rp.Q - r.Q[perm]) < 100 * 1e8 * U_ROUND * math.sqrt(16)


def test_preconditioned_condition_number(ora):
    """Proof of Thm 3.3: kappa_2(W) <= 1.28/(0.8 sqrt((1-eps_s)/(1+eps_b)) - 0.08)
    ~= 6.86 at eps_1 = eps_2 = 0.5.  Probabilistic: soft pin with margin."""
    X = _x(16384, 32, 12, 8)
    for algo in ("slhc3", "sslhc3"):
        r = _run(ora, algo, X, seed=1, stages=True)
        W = ora.trsm_right_upper(X, r.stages["Y"])
        s = np.linalg.svd(W, compute_uv=False)
        assert s[0] / s[-1] < 10.0
        # the sketch, S and Y stages agree with their definitions
        assert rel_fro(r.stages["Y"], ora.trmm_uu(r.stages["S"], r.stages["U"])) == 0.0


def test_paper_family_magnitudes(ora):
    """P:963-1014 (tab:Ok / tab:Rk): SVD-stacked X, m = 20000, n = 50, kappa = 1e12 ->
    orthogonality and absolute residual of order 1e-15 for both algorithms."""
    X = synth.svd_stack(20000, 50, 1e-12, 0).numpy()
    for algo in ("slhc3", "sslhc3"):
        r = _run(ora, algo, X, seed=3, s1=17000, s2=50, s=50, b=400, a=4)
        assert orth_err(r.Q) < 1e-14
        assert np.linalg.norm(r.Q @ r.R - X) < 1e-13


def test_arrowhead_breakdown_is_a_value(ora):
    """SSLHC3 with s1 = 8n on the coherent arrowhead breaks down (SURVEY
    exp3); the breakdown is returned as a stage-tagged error, never as NaNs.  SLHC3
    succeeds with the paper's ~1e-30 orthogonality structure."""
    X = synth.arrowhead(20000, 50, 1e-20).numpy()
    codes = []
    for seed in range(4):
        r = _run(ora, "sslhc3", X, seed=seed, s1=400, s2=100, b=400, raise_on_error=False)
        codes.append(r.info[0])
        if r.info[0]:
            assert r.info[0] in (ora.EBREAKDOWN, ora.ERANKDEF)
    assert any(c != 0 for c in codes)
    r = _run(ora, "slhc3", X, seed=0, s=50, b=400)
    assert orth_err(r.Q) < 1e-13
    assert np.all(np.isfinite(r.R))


def test_nonfinite_input(ora):
    X = _x(256, 8, 4, 0); X[17, 3] = np.inf
    r = _run(ora, "slhc3", X, raise_on_error=False)
    assert r.info == (ora.ENONFINITE, ora.ST_INPUT, 17 * 8 + 3)
