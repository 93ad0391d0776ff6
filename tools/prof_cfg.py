"""Run a BASELINE config a few times (for ncu launch lists / full captures).

  python tools/prof_cfg.py cfg2 [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
X = synth.config_matrix(cfg, device=dev)
plan = rl.Plan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, device=dev)
for _ in range(iters):
    res = plan.run(X)
torch.cuda.synchronize()
print(cfg.name, "info", res.info())
