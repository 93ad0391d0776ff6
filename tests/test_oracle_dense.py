"""Pins for the oracle's dense kernels: SPEC worked examples, LAPACK/scipy,
exact invariants and error values."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import GOLDEN, rel_fro

EX = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


def test_spec_examples(ora):
    assert np.array_equal(ora.gram(np.array(EX["gram"]["X"])), np.array(EX["gram"]["G"]))
    assert np.array_equal(ora.chol(np.array(EX["cholesky"]["G"])), np.array(EX["cholesky"]["R"]))
    assert np.array_equal(np.abs(ora.hqr_r(np.array(EX["hqr"]["A"]))), np.array(EX["hqr"]["R_abs"]))
    Q = ora.trsm_right_upper(np.array(EX["trisolve"]["X"]), np.array(EX["trisolve"]["R"]))
    assert np.array_equal(Q, np.array(EX["trisolve"]["Q"]))


def test_gram_symmetry_and_accuracy(ora):
    A = np.random.default_rng(0).standard_normal((10000, 24))
    G = ora.gram(A)
    assert np.array_equal(G, G.T)
    assert rel_fro(G, A.T @ A) < 1e-14


def test_cholesky_roundtrip_and_breakdown(ora):
    rng = np.random.default_rng(1)
    R0 = np.triu(rng.standard_normal((12, 12))) + 6 * np.eye(12)
    R0 *= np.sign(np.diag(R0))[:, None]
    R = ora.chol(R0.T @ R0)
    assert rel_fro(R, R0) < 1e-13
    assert np.array_equal(np.tril(R, -1), np.zeros_like(R))
    G = np.diag([1.0, 2.0, -1.0, 4.0])
    with pytest.raises(ora.OracleError) as e:
        ora.chol(G, stage=ora.ST_CHOL2)
    assert (e.value.code, e.value.stage, e.value.index) == (ora.EBREAKDOWN, ora.ST_CHOL2, 2)
    G = np.eye(3); G[1, 1] = np.nan
    with pytest.raises(ora.OracleError) as e:
        ora.chol(G)
    assert e.value.index == 1


def test_hqr_vs_lapack(ora):
    A = np.random.default_rng(2).standard_normal((100, 10))
    R = ora.hqr_r(A)
    Rl = np.linalg.qr(A)[1]
    # Householder R is unique up to row signs
    d = np.sign(np.diag(R)) * np.sign(np.diag(Rl))
    assert rel_fro(R, Rl * d[:, None]) < 1e-14
    assert np.array_equal(np.tril(R, -1), np.zeros_like(R))
    # LAPACK dgeqr2 sign convention beta = -sign(alpha)||x||: diag(R) sign opposite to the pivot column's head
    assert np.all(np.sign(np.diag(R))[:1] == -np.sign(A[0, 0]))


def test_hqr_zero_column(ora):
    A = np.random.default_rng(3).standard_normal((20, 4)); A[:, 2] = 0
    with pytest.raises(ora.OracleError) as e:
        ora.hqr_r(A)
    assert (e.value.code, e.value.stage, e.value.index) == (ora.ERANKDEF, ora.ST_HQR, 2)


def test_trsm_vs_scipy_and_singular(ora):
    rng = np.random.default_rng(4)
    T = np.triu(rng.standard_normal((16, 16))) + 4 * np.eye(16)
    A = rng.standard_normal((300, 16))
    out = ora.trsm_right_upper(A, T)
    ref = sla.solve_triangular(T, A.T, trans="T", lower=False).T
    assert rel_fro(out, ref) < 1e-13
    T[5, 5] = 0
    with pytest.raises(ora.OracleError) as e:
        ora.trsm_right_upper(A, T, stage=ora.ST_SOLVE_D)
    assert (e.value.code, e.value.stage, e.value.index) == (ora.ESINGULAR, ora.ST_SOLVE_D, 5)


def test_trmm_upper(ora):
    rng = np.random.default_rng(5)
    A = np.triu(rng.standard_normal((9, 9))); B = np.triu(rng.standard_normal((9, 9)))
    C = ora.trmm_uu(A, B)
    assert rel_fro(C, A @ B) < 1e-15
    assert np.array_equal(np.tril(C, -1), np.zeros((9, 9)))
