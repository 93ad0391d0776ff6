"""The paper's section 5 experiments at GPU speed, through the
library's public API (Plan / MethodPlan) on one GPU.

  python tools/experiments.py applicability [--trials T]   # tab:Ok..tab:Rk2
  python tools/experiments.py robustness [--trials T]      # tab:success1..5

Families (synth/): the stacked SVD matrix, the stacked lower-triangular
matrix, the arrowhead, the sprand-like matrix (SPEC
S:469 reading).  Trials vary the sketch seed (the random part of the method) on a fixed X.
Each line of output is one JSON record; a summary table follows.

Sizes follow the paper: section 5.1 m = 20000, n = 50 with eps1 = 0.5, p1 = 0.6 ->
s1 = (n^2+n)/(eps1^2 p1) = 17000 and s(2) = 50; section 5.3 m = 20000, n = 20,
kappa = 1e12, s1 from p1 in {0.3, 0.4, 0.5, 0.6} -> {5600, 4200, 3360, 2800}, s(2) from
p(2) in {0.1, 0.2, 0.3, 0.4} by the eta = 1 rule (R#12) -> 28 ... 20.
Bounds: orthogonality 6(mn u + n(n+1) u) (eq:ortho2ss P:362, eq:orthoss P:389); residual
Phi (eq:res2ss) for SSLHC3 with eps_s = 0.75, eps_b = 1.25 and Theta
(eq:resss) for SLHC3 with eps = 0.5.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

U = 2.0 ** -53  # unit roundoff


def s_gauss(n: int, eps: float, p: float) -> int:
    """Gaussian sketch size, eta = 1 with natural logs and a floor at n (R#12)."""
    return max(n, math.ceil(math.log(n) * math.log(1.0 / p) / eps ** 2))


def s_count(n: int, eps1: float, p1: float) -> int:
    """CountSketch size of eq:e2: s1 >= (n^2 + n) / (eps1^2 p1)."""
    return math.ceil(round((n * n + n) / (eps1 ** 2 * p1), 9))


def ortho_bound(m: int, n: int) -> float:
    """eq:ortho2ss / eq:orthoss."""
    return 6.0 * (m * n * U + n * (n + 1) * U)


def resid_bound(m: int, n: int, eps_s: float, eps_b: float, norm_x2: float) -> float:
    """Phi of Theorem SSLHC3; with eps_s = eps_b = eps it is Theta of Theorem SLHC3."""
    w = m * n * U + n * (n + 1) * U
    h1 = 5.0 * (1.28 / (0.8 * math.sqrt((1 - eps_s) / (1 + eps_b)) - 0.08)) ** 2 * w
    h2 = 1.0 / (4.0 / (5.0 * math.sqrt(1 + eps_b)) - 0.11 / math.sqrt(1 - eps_s))
    return (1.79 * (1 + h1) + 4.63 * math.sqrt(1 + h1) + 1.41) * h2 / math.sqrt(1 - eps_s) * n * n * U * norm_x2


class Runner:
    """Plans (workspace, outputs) cached per method and size; run() returns the metrics."""

    def __init__(self, device):
        self.dev = device
        self.plans = {}

    def plan(self, method: str, m: int, n: int, s: int = 0, s1: int = 0, s2: int = 0):
        key = (method, m, n, s, s1, s2)
        if key not in self.plans:
            if method in ("slhc3", "sslhc3"):
                self.plans[key] = rl.Plan(method, m, n, s=s, s1=s1, s2=s2, device=self.dev)
            else:
                self.plans[key] = rl.MethodPlan(method, m, n, s1=s1, s2=s2, device=self.dev)
        return self.plans[key]

    def run(self, method: str, X: torch.Tensor, seed: int, s: int = 0, s1: int = 0, s2: int = 0) -> dict:
        m, n = X.shape
        p = self.plan(method, m, n, s, s1, s2)
        p.seed = seed
        res = p.run(X)
        code = res.info()
        out = {"code": code[0], "stage": code[1]}
        if code[0] == 0:
            Q, R = res.Q, res.R
            eye = torch.eye(n, dtype=torch.float64, device=self.dev)
            out["orth"] = torch.linalg.norm(Q.T @ Q - eye).item()
            out["resid"] = torch.linalg.norm(Q @ R - X).item()  # absolute, as the paper
        return out


def _agg(recs, m, n, bound_r):
    ok = [r for r in recs if r["code"] == 0]
    b_o = ortho_bound(m, n)
    return {"trials": len(recs), "breakdowns": len(recs) - len(ok),
            "orth_mean": sum(r["orth"] for r in ok) / len(ok) if ok else None,
            "resid_mean": sum(r["resid"] for r in ok) / len(ok) if ok else None,
            "orth_bound": b_o, "resid_bound": bound_r,
            "exceed": sum(1 for r in ok if r["orth"] > b_o or (bound_r is not None and r["resid"] > bound_r))}


def applicability(runner: Runner, trials: int, emit):
    m, n = 20000, 50
    s = 50  # s(2) = 50
    s1 = s_count(n, 0.5, 0.6)  # 17000
    fams = [("svd", "scholqr3", [1e-10, 1e-12, 1e-14, 1e-16], lambda v: synth.svd_stack(m, n, v, 0, device=runner.dev)),
            ("lowertri", "luc2", [-0.7, -0.8, -0.9, -1.0], lambda v: synth.lower_tri_stack(m, n, v, device=runner.dev)),
            ("arrowhead", "rhc", [1e-15, 1e-20, 1e-25, 1e-30], lambda v: synth.arrowhead(m, n, v, device=runner.dev))]
    rows = []
    for fam, other, params, gen in fams:
        for v in params:
            X = gen(v).contiguous()
            nx = torch.linalg.matrix_norm(X, ord=2).item()
            for method in ("slhc3", "sslhc3", other):
                recs = []
                for k in range(trials if method in ("slhc3", "sslhc3", "rhc") else 1):
                    recs.append(runner.run(method, X, seed=1000 + k, s=s, s1=s1, s2=s))
                bound = (resid_bound(m, n, 0.75, 1.25, nx) if method == "sslhc3" else
                         resid_bound(m, n, 0.5, 0.5, nx) if method == "slhc3" else None)
                rec = {"exp": "applicability", "family": fam, "param": v, "method": method, **_agg(recs, m, n, bound)}
                emit(rec)
                rows.append(rec)
    return rows


def robustness(runner: Runner, trials: int, emit):
    m, n = 20000, 20
    X = synth.sprand(m, n, 0.05, 1e12, 7, device=runner.dev)
    nx = torch.linalg.matrix_norm(X, ord=2).item()
    rows = []
    for p1 in (0.3, 0.4, 0.5, 0.6):  # tab:success1 / tab:success2
        s1 = s_count(n, 0.5, p1)
        recs = [runner.run("sslhc3", X, seed=k, s1=s1, s2=20) for k in range(trials)]
        rec = {"exp": "robustness", "vary": "p1", "param": p1, "s1": s1, "s2": 20, "method": "sslhc3",
               **_agg(recs, m, n, resid_bound(m, n, 0.75, 1.25, nx))}
        emit(rec)
        rows.append(rec)
    for p2 in (0.1, 0.2, 0.3, 0.4):  # tab:success3 .. tab:success5
        s2 = s_gauss(n, 0.5, p2)
        for method in ("slhc3", "sslhc3"):
            s1 = s_count(n, 0.5, 0.6)
            recs = [runner.run(method, X, seed=k, s=s2, s1=s1, s2=s2) for k in range(trials)]
            bound = resid_bound(m, n, 0.75, 1.25, nx) if method == "sslhc3" else resid_bound(m, n, 0.5, 0.5, nx)
            rec = {"exp": "robustness", "vary": "p2", "param": p2, "s": s2, "s1": s1, "method": method,
                   **_agg(recs, m, n, bound)}
            emit(rec)
            rows.append(rec)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["applicability", "robustness", "all"])
    ap.add_argument("--trials", type=int, default=100)
    a = ap.parse_args()
    runner = Runner(torch.device("cuda", 0))
    emit = lambda r: print(json.dumps(r), flush=True)  # noqa: E731
    if a.which in ("applicability", "all"):
        applicability(runner, a.trials, emit)
    if a.which in ("robustness", "all"):
        robustness(runner, a.trials, emit)


if __name__ == "__main__":
    main()
