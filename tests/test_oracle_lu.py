"""Pins for the oracle's row-pivoted LU (PX = LU, P:73/P:279/P:293) under the
tournament contract of DESIGN.md R#3-R#5: GEPP equivalence (scipy/LAPACK pivots),
the SPEC worked example, hand-traced trees, reconstruction bounds, invariances."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import GOLDEN


def _perm_from_scipy(X):
    """Pivot row ids (in pivot order) of LAPACK dgetrf via scipy."""
    P, L, U = sla.lu(X)  # X = P L U
    m, n = X.shape
    order = np.argmax(P, axis=0)   # row k of (P^T X) is X[order[k]]
    return order[:n], U[:n]


def test_spec_example(ora):
    ex = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["lu"]
    piv, U, L11 = ora.tslu(np.array(ex["X"]), leaf_rows=8, arity=2)
    assert list(piv) == ex["piv"]
    assert np.allclose(U, ex["U"], rtol=0, atol=1e-15)
    assert np.allclose(L11, ex["L11"], rtol=0, atol=1e-16)


@pytest.mark.parametrize("m,n,panel", [(300, 12, 12), (257, 40, 40), (500, 33, 8), (129, 64, 16)])
def test_single_leaf_is_gepp(ora, m, n, panel):
    """One leaf (b >= m): tournament == Gaussian elimination with partial pivoting for
    any panel width; pivots equal LAPACK's on tie-free random inputs."""
    X = np.random.default_rng(m + n).standard_normal((m, n))
    piv, U, L11, L = ora.tslu(X, leaf_rows=m, arity=2, panel=panel, want_L=True)
    pl, Ul = _perm_from_scipy(X)
    assert list(piv) == list(pl)
    assert np.linalg.norm(U - Ul) <= 1e-13 * np.linalg.norm(Ul)
    assert np.abs(L).max() <= 1.0   # |L| <= 1 under GEPP


def _hand_tree():
    # m = 8 rows, n = 2, leaves of 2 rows, arity 2.  Column 0 magnitudes chosen so the
    # tournament differs from GEPP; rows 5 and 6 tie in |col 0| (smaller id wins).
    X = np.array([[1.0, 2.0],
                  [3.0, 1.0],
                  [-2.0, 5.0],
                  [0.5, 1.0],
                  [4.0, 4.0],
                  [-6.0, 1.0],
                  [6.0, 2.0],
                  [0.25, 8.0]])
    return X


def test_hand_traced_tree(ora):
    """Hand trace (panel = n = 2, b = 2, arity 2):
    leaves {0,1}->(1,0) ; {2,3}->(2,3) ; {4,5}->(5,4) ; {6,7}->(6,7)
      leaf {0,1}: p=1 (|3|); row0: l=1/3, x01 = 2-1/3*1 = 5/3 -> picks 0.   out (1,0)
      leaf {2,3}: p=2 (|-2|); row3: l=-1/4, 1 - (-1/4)*5 = 2.25 -> out (2,3)
      leaf {4,5}: p=5 (|-6|); row4: l=-2/3, 4-(-2/3)*1 = 14/3 -> out (5,4)
      leaf {6,7}: p=6 (|6|); row7: l=1/24, 8-2/24 -> out (6,7)
    level 1: node {1,0,2,3}: p=1 (|3| > |-2|), updates: row0 5/3, row2 l=-2/3: 5+2/3=17/3, row3 l=1/6: 1-1/6=5/6
               -> col1 max is row2 (17/3) -> out (1,2)
             node {5,4,6,7}: |−6| and |6| tie -> smaller id 5; row4 l=-2/3 -> 14/3; row6 l=-1 -> 2+1=3;
               row7 l=-1/24 -> 8+1/24 -> out (5,7)
    root {1,2,5,7}: p=5 (|-6|); row1 l=-1/2 -> 1+1/2 = 1.5; row2 l=1/3 -> 5-1/3=14/3; row7 l=-1/24 -> 8+1/24
               -> col1 max row7 -> piv (5,7)."""
    X = _hand_tree()
    piv, U, L11 = ora.tslu(X, leaf_rows=2, arity=2)
    assert list(piv) == [5, 7]
    assert U[0, 0] == -6.0 and U[0, 1] == 1.0
    assert abs(U[1, 1] - (8 + 1 / 24)) < 1e-15
    # GEPP on the same matrix picks 5 as well (tie with 6 -> id 5), then row 7
    piv_g, _, _ = ora.tslu(X, leaf_rows=8, arity=2)
    assert list(piv_g) == [5, 7]


def test_tie_break_smallest_id_and_zero_leaf(ora):
    X = np.array([[0.0, 0.0], [0.0, 0.0], [2.0, 1.0], [-2.0, 3.0], [0.0, 0.0], [0.0, 1.0]])
    piv, U, L11 = ora.tslu(X, leaf_rows=2, arity=3)
    # leaf {0,1} is all zero: zero-column rule picks ids 0 then 1 without updates
    assert piv[0] == 2           # |2| == |-2|, smaller id wins
    assert piv[1] == 3           # after elimination row3 col1 = 3+1 = 4 is the largest
    X2 = X.copy(); X2[[2, 3]] = X2[[3, 2]]
    piv2, _, _ = ora.tslu(X2, leaf_rows=2, arity=3)
    assert piv2[0] == 2 and X2[2, 0] == -2.0


def test_reconstruction_and_L_consistency(ora):
    """||PX - LU||_F <= 2 m n u ||X||_F; L from the elimination equals L
    recomputed by forward substitution bit for bit (same fma chain, DESIGN R#O5)."""
    rng = np.random.default_rng(9)
    for (m, n, b, a, panel) in [(4096, 32, 128, 4, 32), (3000, 24, 100, 3, 8), (2048, 16, 64, 8, 16)]:
        X = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -8, n))
        piv, U, L11, L = ora.tslu(X, leaf_rows=b, arity=a, panel=panel, want_L=True)
        assert len(set(piv.tolist())) == n
        err = np.linalg.norm(X - L @ U)   # original row order: X = L U row by row
        assert err <= 2 * m * n * 2 ** -53 * np.linalg.norm(X)
        L2 = ora.lfactor(X, piv, U, L11)
        assert np.array_equal(L, L2)
        assert np.array_equal(L[piv], L11)
        assert np.abs(L).max() < 4.0  # tournament growth stays small (observed 1.2-1.4)


def test_pivots_invariant_to_row_order_inside_leaves(ora):
    """A node's output depends only on its candidate set (id tie-breaks): shuffling rows
    inside each leaf block permutes the ids of the pivots and leaves U unchanged."""
    rng = np.random.default_rng(10)
    m, n, b = 1024, 16, 64
    X = rng.standard_normal((m, n))
    perm = np.concatenate([rng.permutation(np.arange(l, l + b)) for l in range(0, m, b)])
    # rows are re-labelled, so ties are broken differently only if values tie (they do not)
    piv, U, L11 = ora.tslu(X, leaf_rows=b, arity=4)
    piv2, U2, _ = ora.tslu(X[perm], leaf_rows=b, arity=4)
    assert list(perm[piv2]) == list(piv)
    assert np.array_equal(U, U2)


def test_rank_deficient_and_arrowhead(ora):
    import synth
    X = np.random.default_rng(11).standard_normal((500, 6)); X[:, 3] = 0.0
    with pytest.raises(ora.OracleError) as e:
        ora.tslu(X, leaf_rows=50, arity=2)
    assert (e.value.code, e.value.stage, e.value.index) == (ora.ERANKDEF, ora.ST_LU, 3)
    A = synth.arrowhead(2000, 20, 1e-15).numpy()      # 1980 zero rows: zero-column rule
    piv, U, L11, L = ora.tslu(A, leaf_rows=40, arity=4, want_L=True)
    assert np.linalg.norm(A - L @ U) <= 1e-14 * np.linalg.norm(A)
