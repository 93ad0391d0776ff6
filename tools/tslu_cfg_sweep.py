"""TSLU stage time for cfg2 under different tournament contracts (leaf_rows, arity, panel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402
from paper_2412_06551_b200 import _lib  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
X = synth.config_matrix(cfg, device="cuda")
for c in [(256, 4, 64), (512, 16, 32), (512, 8, 32), (512, 32, 16), (512, 16, 16)]:
    plan = rl.Plan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, cfg=c, device="cuda")
    res = plan.run(X)
    torch.cuda.synchronize()
    _lib.lib().rlhc_stage_timing(1)
    _lib.stage_times()
    for _ in range(5):
        res = plan.run(X)
    st = _lib.stage_times()
    _lib.lib().rlhc_stage_timing(0)
    Q = res.Q
    orth = torch.linalg.norm(Q.T @ Q - torch.eye(cfg.n, device="cuda", dtype=torch.float64)).item()
    print(c, "tslu %.1f us" % (1000 * st["tslu"] / st["calls"]), "total %.1f us" %
          (1000 * sum(v for k, v in st.items() if k != "calls") / st["calls"]), "info", res.info(), "orth %.2e" % orth,
          flush=True)
