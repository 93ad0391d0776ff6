"""Seeded synthetic test matrices -- shared input generator for the CUDA path, the
oracle, the tests and bench.py.  Holds none of the method's arithmetic (no Philox,
no sketch, no LU/QR of the method); it only builds inputs X with the structure of
BASELINE.json's configs and of the paper's experiment families (section 5).

Generation uses torch's own seeded generator on the requested device (the same
bytes are then copied to the oracle), so the GPU path never depends on the host
RNG for its input at full size.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Config:
    name: str
    algo: str          # "slhc3" | "sslhc3"
    m: int
    n: int
    s: int = 0         # SLHC3 Gaussian sketch rows
    s1: int = 0        # SSLHC3 CountSketch rows
    s2: int = 0        # SSLHC3 Gaussian rows
    kappa_exp: int = 8 # sigma log-spaced from 1 to 10^-kappa_exp
    colscale: bool = False
    seed: int = 0

    @property
    def sketch_rows(self) -> int:
        return self.s if self.algo == "slhc3" else self.s2


# BASELINE.json "configs" (restated)
CONFIGS = {
    "cfg1": Config("cfg1", "slhc3", 2048, 16, s=32, kappa_exp=8, seed=0),
    "cfg2": Config("cfg2", "slhc3", 65536, 64, s=128, kappa_exp=12, seed=1),
    "cfg3": Config("cfg3", "sslhc3", 1 << 20, 128, s1=1024, s2=256, kappa_exp=15, colscale=True, seed=2),
    "cfg4a": Config("cfg4a", "slhc3", 262144, 512, s=1024, kappa_exp=10, seed=3),
    "cfg4b": Config("cfg4b", "sslhc3", 262144, 512, s1=4096, s2=1024, kappa_exp=10, seed=3),
    "cfg5": Config("cfg5", "sslhc3", 1 << 24, 256, s1=2048, s2=512, kappa_exp=14, seed=4),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + 12345)
    return g


CHUNK = 1 << 16  # rows per independently seeded chunk of A (any aligned row range can be generated alone)


def baseline_matrix(m: int, n: int, kappa_exp: float, seed: int, colscale: bool = False, device="cpu",
                    row0: int = 0, rows: int | None = None) -> torch.Tensor:
    """X = A diag(sigma) V^T (BASELINE.json configs): A iid N(0, 1/m) m x n, V the
    Q factor of an iid N(0,1) n x n matrix, sigma_k = 10^(-kappa_exp k/(n-1)); optional
    column scaling by 10^u, u ~ U[-3, 3] (cfg3).  Rows [row0, row0 + rows) of X (default: all),
    generated on `device`; A's rows come in chunks of CHUNK rows, each from its own seeded
    stream, so a row shard is bitwise the same rows of the full matrix."""
    dev = torch.device(device)
    rows = m - row0 if rows is None else rows
    g = _gen(seed, dev)
    Vg = torch.randn(n, n, generator=g, device=dev, dtype=torch.float64)
    V, Rv = torch.linalg.qr(Vg)
    V = V * torch.sign(torch.diagonal(Rv)).unsqueeze(0)
    k = torch.arange(n, device=dev, dtype=torch.float64)
    sigma = torch.pow(torch.tensor(10.0, device=dev, dtype=torch.float64),
                      -float(kappa_exp) * k / max(n - 1, 1))
    B = sigma.unsqueeze(1) * V.T                    # diag(sigma) V^T
    if colscale:
        u = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 6.0 - 3.0
        B = B * torch.pow(torch.tensor(10.0, device=dev, dtype=torch.float64), u).unsqueeze(0)
    X = torch.empty(rows, n, device=dev, dtype=torch.float64)
    scale = 1.0 / math.sqrt(m)
    c_lo, c_hi = row0 // CHUNK, (row0 + rows + CHUNK - 1) // CHUNK
    for c in range(c_lo, c_hi):
        gc = _gen(seed * 7919 + 1 + c, dev)
        a0, a1 = c * CHUNK, min(m, (c + 1) * CHUNK)
        A = torch.randn(a1 - a0, n, generator=gc, device=dev, dtype=torch.float64) * scale
        lo, hi = max(a0, row0), min(a1, row0 + rows)
        torch.matmul(A[lo - a0:hi - a0], B, out=X[lo - row0:hi - row0])
    return X


def config_matrix(cfg: Config, device="cpu", m: int | None = None) -> torch.Tensor:
    return baseline_matrix(m or cfg.m, cfg.n, cfg.kappa_exp, cfg.seed, cfg.colscale, device=device)


# ---- the paper's experiment families (section 5), for stress tests ----
def svd_stack(m: int, n: int, sigma: float, seed: int, blocks: int = 10, device="cpu") -> torch.Tensor:
    """X = 10 stacked copies of X1 = O Sigma H^T, Sigma = diag(sigma^(k/(n-1)))."""
    dev = torch.device(device); g = _gen(seed, dev)
    mb = m // blocks
    O, _ = torch.linalg.qr(torch.randn(mb, n, generator=g, device=dev, dtype=torch.float64))
    H, _ = torch.linalg.qr(torch.randn(n, n, generator=g, device=dev, dtype=torch.float64))
    k = torch.arange(n, device=dev, dtype=torch.float64)
    S = torch.pow(torch.tensor(sigma, device=dev, dtype=torch.float64), k / (n - 1))
    X1 = (O * S.unsqueeze(0)) @ H.T
    return X1.repeat(blocks, 1)


def lower_tri_stack(m: int, n: int, a: float, device="cpu", diag: float = 1.0) -> torch.Tensor:
    """stacked lower-triangular F (a below the diagonal).  The paper prints 100 on
    the diagonal, but its tables (tab:Ok1/Rk1) give kappa_2(X) = 2.65e12, 5.10e13,
    8.29e14, 1.13e16 for a = -0.7 .. -1, which a unit diagonal reproduces (2.65e12, 5.10e13,
    8.27e14, 1.06e16; with 100 on the diagonal kappa_2 is 1.21 .. 1.33): DESIGN.md R#25."""
    F = torch.full((n, n), float(a), dtype=torch.float64, device=device).tril(-1) + \
        float(diag) * torch.eye(n, dtype=torch.float64, device=device)
    reps = -(-m // n)
    return F.repeat(reps, 1)[:m].contiguous()


def arrowhead(m: int, n: int, beta: float, device="cpu") -> torch.Tensor:
    """X = -5 e1 e1zs^T + [E; 0], E = diag(beta^(k/(n-1)))."""
    X = torch.zeros(m, n, dtype=torch.float64, device=device)
    k = torch.arange(n, dtype=torch.float64, device=device)
    X[:n, :n] = torch.diag(torch.pow(torch.tensor(beta, dtype=torch.float64, device=device), k / (n - 1)))
    X[0, 1:] += -5.0
    return X


def sprand(m: int, n: int, density: float, kappa: float, seed: int, device="cpu") -> torch.Tensor:
    """P:1199 (section 5.3): MATLAB sprand(m, n, density, 1/kappa) stand-in, the SPEC S:469
    reading: a sparse pattern with iid Bernoulli(density) support and N(0,1) values, its
    thin SVD, singular values replaced by the geometric ladder 1 ... 1/kappa, recomposed
    (dense).  The paper does not state sprand's value distribution (SPEC 'Open Questions')."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    vals = torch.randn(m, n, generator=g, device=dev, dtype=torch.float64)
    mask = torch.rand(m, n, generator=g, device=dev, dtype=torch.float64) < density
    S = torch.where(mask, vals, torch.zeros((), dtype=torch.float64, device=dev))
    U, _, Vh = torch.linalg.svd(S, full_matrices=False)
    k = torch.arange(n, device=dev, dtype=torch.float64)
    sig = torch.pow(torch.tensor(1.0 / kappa, dtype=torch.float64, device=dev), k / max(n - 1, 1))
    return ((U * sig.unsqueeze(0)) @ Vh).contiguous()
