"""The row-chunked oracle (ora_lhc3_chunked: X streamed in row chunks, never stored; the
cfg5 oracle, SURVEY 8(c) "processes X in row chunks") against the in-memory oracle
(ora_slhc3 / ora_sslhc3, pinned by test_oracle_*): bit-identical piv, every stage (U, L11,
L_t, L_s, S, Y, G1, D, G2, J), R and every row of Q, on shapes that exercise ragged last
chunks / leaves / Gram blocks, partial tree groups, several panels and chunk sizes, and the
same error values (rank deficiency, non-finite input)."""
import numpy as np
import pytest

import synth


def _chunked(ora, algo, X, a, b, seed, c, chunk):
    m, n = X.shape
    Q = np.full((m, n), np.nan)

    def put(r0, q):
        Q[r0:r0 + len(q)] = q
    res = ora.lhc3_chunked(algo, m, n, lambda r0, rows: X[r0:r0 + rows], a, b, seed, *c, chunk_rows=chunk,
                           put_q=put, stages=True, raise_on_error=False)
    return res, Q


@pytest.mark.parametrize("algo,m,n,a,b,c,chunk", [
    ("sslhc3", 20000, 48, 512, 96, (128, 8, 16), 4096),     # ragged last chunk, 3 panels
    ("sslhc3", 33000, 24, 200, 48, (64, 4, 8), 8192),       # partial groups at every level
    ("sslhc3", 65536, 32, 256, 64, (128, 8, 16), 65536),    # one chunk, complete 8-ary tree
    ("slhc3", 9000, 40, 80, 0, (128, 3, 16), 1024),         # ragged panel (w = 8), 71 leaves
    ("slhc3", 3000, 16, 32, 0, (3000, 2, 16), 24000),       # one leaf: exact GEPP
    ("slhc3", 12345, 20, 40, 0, (64, 2, 16), 192),          # many small chunks, deep binary tree
])
def test_chunked_equals_in_memory(ora, algo, m, n, a, b, c, chunk):
    X = synth.baseline_matrix(m, n, 10, 3).numpy()
    ref = (ora.sslhc3(X, a, b, 7, *c, stages=True) if algo == "sslhc3"
           else ora.slhc3(X, a, 7, *c, stages=True))
    res, Q = _chunked(ora, algo, X, a, b, 7, c, chunk)
    assert res.info == (0, 0, 0)
    assert np.array_equal(ref.piv, res.piv)
    for k in ref.stages:
        assert np.array_equal(ref.stages[k], res.stages[k]), k
    assert np.array_equal(ref.R, res.R)
    assert np.array_equal(ref.Q, Q)


def test_chunked_error_values(ora):
    rng = np.random.default_rng(3)
    m, n = 4096, 16
    X = rng.standard_normal((m, n))
    X[:, 5] = 0.0  # rank deficient: the root finds an exactly zero pivot column
    ref = ora.sslhc3(X, 256, 32, 1, 128, 8, 16, raise_on_error=False)
    res, _ = _chunked(ora, "sslhc3", X, 256, 32, 1, (128, 8, 16), 1024)
    assert ref.info[0] == ora.ERANKDEF and res.info == ref.info
    X = rng.standard_normal((m, n))
    X[3001, 7] = np.inf
    ref = ora.slhc3(X, 32, 1, 128, 8, 16, raise_on_error=False)
    res, _ = _chunked(ora, "slhc3", X, 32, 0, 1, (128, 8, 16), 1024)
    assert ref.info[0] == ora.ENONFINITE and res.info == ref.info
    # chunks must hold whole leaves and whole 64-row Gram blocks
    res, _ = _chunked(ora, "slhc3", rng.standard_normal((m, n)), 32, 0, 1, (128, 8, 16), 1000)
    assert res.info[0] == ora.EINVAL
