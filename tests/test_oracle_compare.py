"""Pins of the oracle's comparison algorithms: CholeskyQR2 (alg:cholqr2,
P:36-46), SCholeskyQR3 (alg:Shifted3, shift of P:984), LUC2 (alg:LU2) and
RHC (alg:Rand2), against things other than themselves:
  * the thin QR with diag(R) > 0 is unique, so every method's R must equal LAPACK's
    (sign-normalised) on a well-conditioned X, with orthogonal Q and a small residual;
  * X = [I; 0] gives Q = X, R = I exactly (every Gram / Cholesky / substitution is exact;
    RHC to rounding, its Householder R of a Gaussian sketch is not exact);
  * the applicability claims of the paper: CholeskyQR2 "is inapplicable ... to deal with
    ill-conditioned matrices" -- it breaks down in its first Cholesky once
    kappa^2 u > 1; SCholeskyQR3 extends the range; LUC2 "has no requirement on
    kappa_2(X)" and RHC succeeds on ill-conditioned X -- both at kappa = 1e15;
  * column scaling: R(X D) = R(X) D for a positive diagonal D (uniqueness of the thin QR)."""
import math

import numpy as np
import pytest

import synth
from conftest import qr_signed, rel_fro

METHODS = {
    "cholqr2": lambda ora, X: ora.cholqr2(X, raise_on_error=False),
    "scholqr3": lambda ora, X: ora.scholqr3(X, raise_on_error=False),
    "luc2": lambda ora, X: ora.luc2(X, 512, 16, None, raise_on_error=False),
    "rhc": lambda ora, X: ora.rhc(X, min(X.shape[0], 8 * X.shape[1]), 2 * X.shape[1], 3, raise_on_error=False),
}


@pytest.mark.parametrize("name", sorted(METHODS))
def test_unique_qr(ora, name):
    rng = np.random.default_rng(7)
    X = rng.standard_normal((3000, 40)) @ np.diag(np.logspace(0, -3, 40))
    res = METHODS[name](ora, X)
    assert res.info == (0, 0, 0)
    Q0, R0 = qr_signed(X)
    assert np.all(np.diag(res.R) > 0)
    assert np.array_equal(np.tril(res.R, -1), np.zeros_like(res.R))
    assert rel_fro(res.R, R0) <= 1e-13
    assert ora.orthogonality(res.Q) <= 1e-14 * math.sqrt(40) * 10
    assert ora.residual(res.Q, res.R, X) <= 1e-15 * 40 * 10


@pytest.mark.parametrize("name", sorted(METHODS))
def test_identity(ora, name):
    n, m = 12, 96
    X = np.zeros((m, n))
    X[:n, :n] = np.eye(n)
    if name == "rhc":
        # the Householder R of the Gaussian sketch carries rounding: close to (X, I), not equal
        res = ora.rhc(X, m, 2 * n, 1)  # s1 = m: no CountSketch collisions (cf. the SSLHC3 pin)
        assert res.info == (0, 0, 0)
        assert np.abs(res.R - np.eye(n)).max() <= 1e-14
        assert np.abs(res.Q - X).max() <= 1e-14
        return
    res = METHODS[name](ora, X)
    assert res.info == (0, 0, 0)
    assert np.array_equal(res.R, np.eye(n))
    assert np.array_equal(res.Q, X)


@pytest.mark.parametrize("kexp", [10, 12])
def test_cholqr2_breaks_down_when_ill_conditioned(ora, kexp):
    X = synth.baseline_matrix(4096, 32, kexp, 11).numpy()
    res = ora.cholqr2(X, raise_on_error=False)
    assert res.info[:2] == (ora.EBREAKDOWN, ora.ST_CHOL0)


def test_scholqr3_extends_the_range(ora):
    X = synth.baseline_matrix(4096, 32, 12, 11).numpy()
    res = ora.scholqr3(X)
    assert res.info == (0, 0, 0)
    assert ora.orthogonality(res.Q) <= 1e-13 * math.sqrt(32)


@pytest.mark.parametrize("name", ["luc2", "rhc"])
def test_luc2_rhc_at_kappa_1e15(ora, name):
    X = synth.baseline_matrix(4096, 32, 15, 11).numpy()
    res = METHODS[name](ora, X)
    assert res.info == (0, 0, 0)
    assert ora.orthogonality(res.Q) <= 1e-13 * math.sqrt(32)
    assert ora.residual(res.Q, res.R, X) <= 1e-14 * 32


@pytest.mark.parametrize("name", sorted(METHODS))
def test_column_scaling(ora, name):
    rng = np.random.default_rng(9)
    X = rng.standard_normal((2048, 24))
    d = 10.0 ** rng.uniform(-2, 2, 24)
    r1 = METHODS[name](ora, X)
    r2 = METHODS[name](ora, X * d)
    assert r1.info == r2.info == (0, 0, 0)
    assert rel_fro(r2.R, r1.R * d) <= 1e-12
