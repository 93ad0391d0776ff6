"""Arrowhead, beta = 1e-25: W = X Y^{-1} by row substitution with and without fma
and with division or reciprocal (exact fma emulated with fractions) -- which op choice blows up."""
import numpy as np, scipy.linalg as sl, sys
from fractions import Fraction
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle, synth
X = synth.arrowhead(20000, 50, 1e-25).numpy()
piv, U, L11, L = oracle.tslu(X, 128, 8, 16, want_L=True)
Ls = oracle.omega_block(1000, 0, 50, 0, 20000) @ L
S = np.linalg.qr(Ls, mode="r"); S = S * (np.sign(np.diag(S)) * np.sign(np.diag(U)))[:, None]
Y = S @ U
Xs = X[:50]
def fma(a, b, c): return float(Fraction(a) * Fraction(b) + Fraction(c))
def subst(use_fma, use_rcp):
    W = np.zeros_like(Xs)
    rd = [1.0 / Y[k, k] for k in range(50)]
    for i in range(50):
        o = W[i]
        for k in range(50):
            acc = Xs[i, k]
            for j in range(k):
                acc = fma(-o[j], Y[j, k], acc) if use_fma else acc - o[j] * Y[j, k]
            o[k] = acc * rd[k] if use_rcp else acc / Y[k, k]
    return W
Wn = sl.solve_triangular(Y.T, Xs.T, lower=True).T
for f in (False, True):
    for r in (False, True):
        W = subst(f, r)
        G = W.T @ W
        try: np.linalg.cholesky(G); ok = 'ok'
        except Exception: ok = 'BREAKDOWN'
        print(f"fma={f} rcp={r}: |W|max {np.abs(W).max():.3e}  rel diff vs LAPACK {np.linalg.norm(W-Wn)/np.linalg.norm(Wn):.3e}  chol {ok}")
