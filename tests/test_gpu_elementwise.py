"""Element-by-element error bounds for the floating-point stages whose parity elsewhere is
normwise: every entry of the GPU result must lie within the
textbook rounding-error bound of that entry, so a kernel that got a few small entries wrong
(a tiny singular direction of G, one row of S) fails here even when the norm does not move.

u = 2^-53, gamma_k = k u / (1 - k u) (Higham, Accuracy and Stability of Numerical Algorithms,
Lemma 3.1).  Two computations of the same quantity that are each within gamma_k |.| of the
exact value differ by at most 2 gamma_k |.|.  Sizes up to n = 512 (cfg4's width).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

U = 2.0 ** -53
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def rl():
    import paper_2412_06551_b200 as rl
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return rl


def gamma(k):
    return k * U / (1.0 - k * U)


def _within(got, ref, bound):
    """Every entry within its bound -- and the check has teeth: moving the entry with the
    smallest bound by 10x that bound (a wrong small entry, normwise invisible) fails it."""
    ok = bool(np.all(np.abs(got - ref) <= bound))
    k = np.unravel_index(np.argmin(bound), bound.shape)
    bad = got.copy()
    bad[k] += 10 * bound[k] + 1e-300
    assert not np.all(np.abs(bad - ref) <= bound)
    return ok


def _randn(shape, seed):
    g = torch.Generator(DEV).manual_seed(seed)
    return torch.randn(*shape, dtype=torch.float64, device=DEV, generator=g)


@pytest.mark.parametrize("rows,n,s,row0", [(3000, 16, 32, 0), (10000, 64, 128, 100), (4000, 512, 1024, 7)])
def test_sketch_gauss_elementwise(rl, ora, rows, n, s, row0):
    """Y = Omega A: |Y_gpu - Omega A| <= gamma_rows (|Omega| |A|) per entry for
    each of the GPU and the oracle's fp64 product (any summation order), so their difference
    is within 2 gamma_rows (|Omega| |A|)."""
    A = _randn((rows, n), rows + n)
    out = rl.sketch_gauss(A, s, 11, 0, row0=row0).cpu().numpy()
    Ah = A.cpu().numpy()
    Om = ora.omega_block(11, 0, s, row0, rows)
    ref = Om @ Ah
    bound = 2 * gamma(rows) * (np.abs(Om) @ np.abs(Ah))
    assert _within(out, ref, bound)


@pytest.mark.parametrize("rows,n", [(100000, 64), (3333, 130), (20000, 256), (20000, 512),
                                    # syrk_tma_kernel (n <= 256): ragged row chunks, n not a
                                    # multiple of 8 or 16, fewer rows than one chunk
                                    (100003, 40), (70001, 200), (29, 8), (65537, 128), (1000, 250)])
def test_gram_elementwise(rl, rows, n):
    """G = A^T A: |G_gpu - A^T A| <= 2 gamma_rows (|A|^T |A|) per entry; G exactly
    symmetric."""
    A = _randn((rows, n), 7 * n)
    G = rl.gram(A)
    assert torch.equal(G, G.T)
    Ah = A.cpu().numpy()
    ref = Ah.T @ Ah
    bound = 2 * gamma(rows) * (np.abs(Ah).T @ np.abs(Ah))
    assert _within(G.cpu().numpy(), ref, bound)


@pytest.mark.parametrize("rows,n", [(4000, 16), (7000, 64), (1500, 200), (2000, 512),
                                    # tri_tma_kernel (64 < n <= 256, >= 8 row tiles per SM):
                                    # ragged last tile, n off the fragment grid
                                    (160001, 72), (300007, 128), (90001, 200)])
def test_trsm_elementwise(rl, ora, rows, n):
    """out = A T^{-1} by substitution and by the explicit inverse (R#9).
    Substitution: each row of out is a forward substitution, so out (T + dT) = A with
    |dT| <= gamma_n |T| (Higham Thm 8.5): |out T - A| <= gamma_n |out| |T| per entry.
    Explicit inverse: out = fl(A X) with X = fl(T^{-1}), |X T - I| <= c gamma_n |X| |T|
    (the inverse by substitution) and the product's own |E| <= gamma_n |A| |X|, so
    |out T - A| <= (c + 1) gamma_n |A| |T^{-1}| |T| per entry.  The numpy evaluation of
    out T adds up to gamma_n |out| |T|.  (Where the oracle's operation order is the contract --
    n <= 64 and the wide substitution -- test_gpu_parity checks bitwise equality.)"""
    A = _randn((rows, n), rows)
    g = torch.Generator(DEV).manual_seed(n)
    T = torch.triu(torch.randn(n, n, dtype=torch.float64, device=DEV, generator=g)) + 4 * torch.eye(
        n, device=DEV, dtype=torch.float64)
    Ah, Th = A.cpu().numpy(), T.cpu().numpy()
    Tinv = np.linalg.inv(Th)
    absAT = np.abs(Ah) @ np.abs(Tinv) @ np.abs(Th)
    for mode in (rl.RLHC_SUBST, rl.RLHC_INV_GEMM):
        out, G, info = rl.trsm_apply(A, T, mode=mode, want_gram=True)
        assert info[0] == 0
        o = out.cpu().numpy()
        # the residual itself is evaluated in fp64 by numpy: allow its own gamma_n |o||T|
        res = np.abs(o @ Th - Ah)
        if mode == rl.RLHC_SUBST:
            bound = 2 * gamma(n + 1) * (np.abs(o) @ np.abs(Th)) + 2 * U * np.abs(Ah)
        else:
            bound = 4 * gamma(n + 1) * absAT + 2 * gamma(n + 1) * (np.abs(o) @ np.abs(Th))
        assert np.all(res <= bound), (mode, float((res / np.maximum(bound, 1e-300)).max()))
        # the fused Gram of the output, element by element (as test_gram_elementwise)
        gb = 2 * gamma(rows) * (np.abs(o).T @ np.abs(o))
        assert _within(G.cpu().numpy(), o.T @ o, gb)


@pytest.mark.parametrize("s,n", [(32, 16), (128, 64), (256, 128), (96, 40), (1024, 512)])
def test_hqr_elementwise(rl, s, n):
    """[H, S] = HouseholderQR(L_s): Householder QR is column-wise backward stable,
    L_s + dL = H S with H orthogonal and ||dL e_j|| <= gamma_cs ||L_s e_j|| (Higham Thm 19.4,
    c a small constant), so per entry |(S^T S - L_s^T L_s)_ij| <= 3 gamma_cs ||L_i|| ||L_j||."""
    A = _randn((s, n), s * n)
    S, info = rl.hqr_r(A)
    assert info[0] == 0
    Sh, Ah = S.cpu().numpy(), A.cpu().numpy()
    assert np.array_equal(np.tril(Sh, -1), np.zeros_like(Sh))
    cn = np.linalg.norm(Ah, axis=0)
    bound = 3 * gamma(8 * s * n) * np.outer(cn, cn)
    assert _within(Sh.T @ Sh, Ah.T @ Ah, bound)


@pytest.mark.parametrize("n", [16, 40, 64, 110])
def test_cholesky_elementwise(rl, n):
    """R = chol(G): the computed R satisfies R^T R = G + dG with |dG| <= gamma_{n+1}
    |R^T| |R| per entry (Higham Thm 10.3); the check's own product adds gamma_n |R^T||R|."""
    A = _randn((4 * n, n), n)
    G = A.T @ A
    Rm, info = rl.cholesky(G)
    assert info[0] == 0
    R, Gh = Rm.cpu().numpy(), G.cpu().numpy()
    bound = 2 * gamma(n + 1) * (np.abs(R).T @ np.abs(R))
    assert _within(R.T @ R, Gh, bound)
