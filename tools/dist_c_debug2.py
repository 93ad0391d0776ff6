"""Debug helper: the test's call sequence on one plan."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_06551_b200 as rl  # noqa: E402
from paper_2412_06551_b200._lib import TsluCfg  # noqa: E402
from paper_2412_06551_b200.dist import CDistPlan  # noqa: E402

m, n = 65536, 64
X = synth.baseline_matrix(m, n, 12, 8, device="cuda")
cfg = TsluCfg(256, 4, 64)
plan = CDistPlan("slhc3", m, n, s=128, seed=3, cfg=cfg, device="cuda")
print("1", plan.run(X).info(), flush=True)
single = rl.slhc3(X, s=128, seed=3, cfg=cfg)
print("2", single.info(), flush=True)
Xd = X.clone()
Xd[:, 5] = 0.0
print("3", plan.run(Xd).info(), flush=True)
Xd[777, 3] = float("nan")
print("4", plan.run(Xd).info(), flush=True)
