"""The row-sharded C entry point (rlhc_sslhc3_dist / rlhc_slhc3_dist) with one NCCL rank on a
config, timed against the single-GPU entry point on the same X: the per-rank cost of the
distributed orchestration (what each rank of a multi-GPU run executes, minus the network).

  python tools/time_dist1.py cfg5 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402
from paper_2412_06551_b200.dist import CDistPlan, NcclComm  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
X = synth.config_matrix(cfg, device=dev)


def timed(f):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


single = rl.Plan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, device=dev)
t1 = timed(lambda: single.run(X))
r1 = single.run(X)
piv1 = r1.piv.clone()
del single, r1
torch.cuda.empty_cache()
plan = CDistPlan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, device=dev, comm=NcclComm())
t2 = timed(lambda: plan.run(X))
out = plan.run(X)
same = torch.equal(plan.piv, piv1)
print(f"{cfg.name}: single-GPU entry {t1:.3f} ms, row-sharded entry (1 NCCL rank) {t2:.3f} ms, pivots equal: {same}")
