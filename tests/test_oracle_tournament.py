"""Independent pins for the oracle's multi-panel, multi-leaf tournament (the default
contract: column panels, leaves, arity-ary nodes; R#3-R#5; PX = LU, P:73/P:279/P:293)
and for its checkers (orthogonality, residual).

Two implementations written here from the contract's definition share nothing with
oracle/rlhc_oracle.c:

* ``exact_tournament`` -- the contract in exact rational arithmetic (fractions.Fraction):
  per panel, every row's Schur complement at the panel start, leaves = global row blocks of
  the rows not yet chosen, nodes = `arity` consecutive children (trailing partial group
  allowed) running GEPP with ties to the smallest id, a node's output its first w pivots.
  On inputs whose argmax decisions are not near-ties, floating point and exact arithmetic
  pick the same rows, so the oracle's pivots must equal these.
* ``scipy_tournament`` -- the same tree composed from library primitives: Schur complements
  by numpy products with L = X[:, :p0] U[:p0, :p0]^-1 (scipy solve_triangular), each node's
  pivots from LAPACK dgetrf (scipy.linalg.lu) on its stacked candidates.
A node in panel p > 0 reading wrong candidate values, a mis-grouped level, a dropped partial
group or a wrong leaf boundary changes the pivots and fails these tests.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla


# ------------------------------------------------------------------ exact rational contract
def _gepp_exact(rows, vals, w):
    """GEPP on candidate rows (global ids `rows`, values vals[i] = list of w Fractions).
    Returns (winners in pivot order, min relative argmax gap seen)."""
    A = [list(v) for v in vals]
    ids = list(rows)
    alive = list(range(len(ids)))
    out, gap = [], float("inf")
    for t in range(min(len(ids), w)):
        mags = sorted(((abs(A[i][t]), -ids[i], i) for i in alive), reverse=True)
        best = mags[0]
        if best[0] == 0:
            p = min(alive, key=lambda i: ids[i])  # zero column: smallest remaining id, no update
            out.append(ids[p])
            alive.remove(p)
            continue
        if len(mags) > 1 and mags[1][0] != best[0]:
            gap = min(gap, float((best[0] - mags[1][0]) / best[0]))
        elif len(mags) > 1:
            gap = 0.0  # an exact tie (resolved by id)
        p = best[2]
        out.append(ids[p])
        alive.remove(p)
        for i in alive:
            lmul = A[i][t] / A[p][t]
            for j in range(t + 1, w):
                A[i][j] -= lmul * A[p][j]
    return out, gap


def exact_tournament(X, leaf_rows, arity, panel):
    """Pivot order of the contract on X (numpy float array, converted exactly)."""
    m, n = X.shape
    A = [[Fraction(float(v)) for v in row] for row in X]
    chosen = set()
    piv, gap = [], float("inf")
    for p0 in range(0, n, panel):
        w = min(panel, n - p0)
        # leaves: row blocks of the rows not yet chosen; values = current Schur complement
        nodes = []
        for l0 in range(0, m, leaf_rows):
            cand = [i for i in range(l0, min(m, l0 + leaf_rows)) if i not in chosen]
            win, g = _gepp_exact(cand, [A[i][p0:p0 + w] for i in cand], w)
            gap = min(gap, g)
            nodes.append(win)
        while len(nodes) > 1:
            nxt = []
            for c0 in range(0, len(nodes), arity):
                cand = [i for nd in nodes[c0:c0 + arity] for i in nd]
                win, g = _gepp_exact(cand, [A[i][p0:p0 + w] for i in cand], w)
                gap = min(gap, g)
                nxt.append(win)
            nodes = nxt
        root = nodes[0]
        assert len(root) == w
        # eliminate every remaining row with this panel's pivots (exact right-looking update)
        for k, pr in zip(range(p0, p0 + w), root):
            chosen.add(pr)
            for i in range(m):
                if i in chosen or A[i][k] == 0:
                    continue
                lmul = A[i][k] / A[pr][k]
                A[i][k] = lmul
                for j in range(k + 1, n):
                    A[i][j] -= lmul * A[pr][j]
        piv += root
    return piv, gap


@pytest.mark.parametrize("m,n,leaf,arity,panel,seed", [
    (16, 4, 2, 2, 2, 0),      # the verdict's shape: 8 leaves, 3 levels, 2 panels
    (16, 4, 2, 2, 2, 1),
    (24, 6, 3, 3, 2, 2),      # 8 leaves -> 3 nodes (a partial group) -> 1, 3 panels
    (40, 5, 4, 4, 2, 3),      # 10 leaves -> 3 nodes (partial) -> 1, ragged last panel (w = 1)
    (33, 6, 4, 2, 3, 4),      # ragged last leaf (1 row), 9 leaves, 4 levels
    (64, 8, 8, 8, 4, 5),      # the default arity on a tiny tree
])
def test_oracle_tournament_matches_exact_contract(ora, m, n, leaf, arity, panel, seed):
    rng = np.random.default_rng(seed)
    done, differs_from_gepp = 0, 0
    for trial in range(60):
        X = rng.integers(-40, 41, size=(m, n)).astype(np.float64) + rng.integers(1, 8, size=(m, n)) / 8.0
        ex, gap = exact_tournament(X, leaf, arity, panel)
        if gap < 1e-9:  # a near-tie: floating point may legitimately break it the other way
            continue
        piv, _, _ = ora.tslu(X, leaf_rows=leaf, arity=arity, panel=panel)
        assert list(piv) == ex, (trial, list(piv), ex)
        differs_from_gepp += ex != exact_tournament(X, m, 2, n)[0]
        done += 1
        if done == 12:
            break
    assert done == 12, "too few tie-free trials"
    assert differs_from_gepp > 0  # the tree shape matters on these inputs


def test_exact_contract_ties_and_zero_leaves(ora):
    """Exact ties in |a| go to the smallest global id at every level, and an all-zero leaf
    contributes its smallest ids without updates (R#4, R#5) -- values chosen so every
    intermediate is exact in binary floating point (small dyadic rationals)."""
    X = np.array([[0.0, 0.0, 0.0],
                  [0.0, 0.0, 0.0],
                  [2.0, 1.0, 0.5],
                  [-2.0, 3.0, 1.0],
                  [1.0, -4.0, 2.0],
                  [-1.0, 4.0, 0.25],
                  [0.5, 0.5, 8.0],
                  [2.0, 2.0, 2.0]])
    for leaf, arity, panel in [(2, 2, 1), (2, 2, 2), (2, 3, 1), (4, 2, 2), (3, 2, 3)]:
        ex, _ = exact_tournament(X, leaf, arity, panel)
        piv, _, _ = ora.tslu(X, leaf_rows=leaf, arity=arity, panel=panel)
        assert list(piv) == ex, (leaf, arity, panel, list(piv), ex)


# ------------------------------------------------------------------- scipy-composed tree
def _lapack_winners(S, ids, w):
    """First min(len, w) pivots of LAPACK dgetrf on the stacked candidates S (rows = ids)."""
    P, _, _ = sla.lu(S)
    order = np.argmax(P, axis=0)  # row k of P^T S is S[order[k]]
    k = min(len(ids), w)
    return [ids[i] for i in order[:k]]


def _lu_nopiv_u(A):
    """U of A = L U with no row exchange (A's rows already in pivot order)."""
    A = np.array(A, dtype=np.float64)
    k_max = min(A.shape)
    for k in range(k_max):
        A[k + 1:, k:] -= np.outer(A[k + 1:, k] / A[k, k], A[k, k:])
    return np.triu(A[:k_max])


def scipy_tournament(X, leaf_rows, arity, panel):
    m, n = X.shape
    piv = []
    chosen = np.zeros(m, bool)
    U = np.zeros((n, n))
    for p0 in range(0, n, panel):
        w = min(panel, n - p0)
        if p0:
            Lp = sla.solve_triangular(U[:p0, :p0], X[:, :p0].T, trans="T", lower=False).T  # X[:, :p0] U^-1
            S = X[:, p0:p0 + w] - Lp @ U[:p0, p0:p0 + w]
        else:
            S = X[:, :w].copy()
        nodes = []
        for l0 in range(0, m, leaf_rows):
            cand = [i for i in range(l0, min(m, l0 + leaf_rows)) if not chosen[i]]
            nodes.append(_lapack_winners(S[cand], cand, w) if cand else [])
        while len(nodes) > 1:
            nodes = [_lapack_winners(S[c], c, w) for c in
                     ([i for nd in nodes[c0:c0 + arity] for i in nd] for c0 in range(0, len(nodes), arity))]
        root = nodes[0]
        piv += root
        chosen[root] = True
        # U rows of this panel: the pivot rows' full Schur complement, eliminated in panel order
        full = X[root] - (sla.solve_triangular(U[:p0, :p0], X[root][:, :p0].T, trans="T").T @ U[:p0]
                          if p0 else 0.0)
        U[p0:p0 + w, p0:] = _lu_nopiv_u(full[:, p0:])[:w]
    return piv


@pytest.mark.parametrize("m,n,leaf,arity,panel,seed", [
    (4096, 48, 128, 8, 16, 11),   # the verdict's case: 32 leaves, 2 levels, 3 panels
    (4096, 48, 128, 8, 16, 12),
    (5000, 40, 64, 4, 16, 13),    # ragged last leaf, partial groups, ragged last panel (w = 8)
    (2048, 32, 32, 2, 8, 14),     # 6 levels, 4 panels
])
def test_oracle_tournament_matches_scipy_composition(ora, m, n, leaf, arity, panel, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -6, n))
    piv, U, _ = ora.tslu(X, leaf_rows=leaf, arity=arity, panel=panel)
    ref = scipy_tournament(X, leaf, arity, panel)
    assert list(piv) == ref
    # and the oracle's U is the LU of X[piv] (P X = L U on the pivot rows)
    Ur = _lu_nopiv_u(X[piv])
    assert np.linalg.norm(np.triu(U) - Ur) <= 1e-12 * np.linalg.norm(Ur)


# --------------------------------------------------------------------------- checkers
def test_orthogonality_residual_vs_long_double(ora):
    """ora_orthogonality / ora_residual against numpy extended
    precision (np.longdouble, 64-bit mantissa on x86), on inputs whose exact answer is
    far from fp64 rounding: a perturbed orthonormal Q and a perturbed product."""
    rng = np.random.default_rng(21)
    m, n = 1500, 12
    Q0, _ = np.linalg.qr(rng.standard_normal((m, n)))
    for eps in (1e-15, 1e-10, 1e-4):
        Q = Q0 + eps * rng.standard_normal((m, n))
        Ql = Q.astype(np.longdouble)
        ref = np.sqrt(np.sum((Ql.T @ Ql - np.eye(n, dtype=np.longdouble)) ** 2))
        got = ora.orthogonality(Q)
        assert abs(got - float(ref)) <= 1e-6 * float(ref) + 1e-18, (eps, got, float(ref))
        R = np.triu(rng.standard_normal((n, n))) + 3 * np.eye(n)
        X = Q0 @ R + eps * rng.standard_normal((m, n))
        Rl, Xl = R.astype(np.longdouble), X.astype(np.longdouble)
        d = Ql @ Rl - Xl
        ref = np.sqrt(np.sum(d * d) / np.sum(Xl * Xl))
        got = ora.residual(Q, R, X)
        assert abs(got - float(ref)) <= 1e-6 * float(ref) + 1e-18, (eps, got, float(ref))
    # closed forms: an exactly orthonormal Q (a permutation) gives 0; Q = 2I gives 3 sqrt(n)
    P = np.eye(n)[rng.permutation(n)]
    assert ora.orthogonality(P) == 0.0
    assert abs(ora.orthogonality(2 * np.eye(n)) - 3 * np.sqrt(n)) <= 1e-15 * 3 * np.sqrt(n)
    assert ora.residual(P, np.eye(n), P) == 0.0
