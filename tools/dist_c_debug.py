"""Debug helper: one CDistPlan run on one GPU.  args: algo m n s_or_s1 s2 arity [rankdef]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_06551_b200._lib import TsluCfg  # noqa: E402
from paper_2412_06551_b200.dist import CDistPlan  # noqa: E402

algo, m, n, s1, s2, arity = sys.argv[1], *map(int, sys.argv[2:7])
X = synth.baseline_matrix(m, n, 12, 8, device="cuda")
if len(sys.argv) > 7:
    X[:, 5] = 0.0
if len(sys.argv) > 8:
    X[777, 3] = float("nan")
kw = dict(s=s1) if algo == "slhc3" else dict(s1=s1, s2=s2)
plan = CDistPlan(algo, m, n, seed=3, cfg=TsluCfg(256, arity, 64), device="cuda", **kw)
res = plan.run(X)
torch.cuda.synchronize()
print(sys.argv[1:], "info", res.info(), flush=True)
