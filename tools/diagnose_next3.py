"""NEXT-3 diagnosis: breakdown rates of the paper's applicability
families under both pivot contracts, on the GPU and in the oracle, next to the paper's tables.

  python tools/diagnose_next3.py [--trials 200] [--oracle-trials 40]

Families (section 5, m = 20000, n = 50): the stacked lower-triangular matrix
(a in {-0.7, -0.8, -0.9, -1}) and the arrowhead (beta in {1e-15,
1e-20, 1e-25, 1e-30}).  Methods: SLHC3 (s = 50), SSLHC3 (s1 = 17000, s2 = 50), LUC2.
Pivot contracts: the tournament (128-row leaves, 8-ary nodes, 16-column panels; R#3)
and exact partial pivoting (one leaf of all m rows = LAPACK's GEPP, the paper's MATLAB lu).
Trials vary the sketch seed on a fixed X; one JSON line per (family, param, method, contract,
side) with the breakdown count and the stage of the first failure; a failure must be a
reported EBREAKDOWN (no NaN in a returned Q).
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

M, N, S, S1 = 20000, 50, 50, 17000


def contract(mode):
    return (128, 8, 16) if mode == "tournament" else (M, 2, 16)


def gpu_runs(method, X, mode, trials):
    dev = X.device
    c = contract(mode)
    if method in ("slhc3", "sslhc3"):
        plan = rl.Plan(method, M, N, s=S, s1=S1, s2=S, cfg=c, device=dev)
    else:
        plan = rl.MethodPlan("luc2", M, N, cfg=c, device=dev)
        trials = 1  # LUC2 is deterministic
    codes = []
    for k in range(trials):
        plan.seed = 1000 + k
        res = plan.run(X)
        code = res.info()
        if code[0] == 0:
            assert torch.isfinite(res.Q).all().item(), "a success with non-finite Q"
        codes.append(code)
    return codes


def oracle_runs(method, Xh, mode, trials):
    c = contract(mode)
    codes = []
    for k in range(trials if method != "luc2" else 1):
        if method == "slhc3":
            r = oracle.slhc3(Xh, S, 1000 + k, *c, raise_on_error=False)
        elif method == "sslhc3":
            r = oracle.sslhc3(Xh, S1, S, 1000 + k, *c, raise_on_error=False)
        else:
            r = oracle.luc2(Xh, *c, raise_on_error=False)
        codes.append(r.info)
    return codes


def summary(codes):
    fails = [c for c in codes if c[0] != 0]
    stages = collections.Counter(f"{c[0]}/{c[1]}" for c in fails)
    return {"trials": len(codes), "breakdowns": len(fails), "codes": dict(stages)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=200)
    ap.add_argument("--oracle-trials", type=int, default=40)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    fams = [("lowertri", [-0.7, -0.8, -0.9, -1.0], lambda v: synth.lower_tri_stack(M, N, v, device=dev)),
            ("arrowhead", [1e-15, 1e-20, 1e-25, 1e-30], lambda v: synth.arrowhead(M, N, v, device=dev))]
    for fam, params, gen in fams:
        for v in params:
            X = gen(v).contiguous()
            Xh = np.ascontiguousarray(X.cpu().numpy())
            for method in ("slhc3", "sslhc3", "luc2"):
                for mode in ("tournament", "gepp"):
                    g = summary(gpu_runs(method, X, mode, args.trials))
                    o = summary(oracle_runs(method, Xh, mode, args.oracle_trials))
                    print(json.dumps({"family": fam, "param": v, "method": method, "pivot": mode, "gpu": g,
                                      "oracle": o}), flush=True)


if __name__ == "__main__":
    main()
