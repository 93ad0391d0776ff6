"""Time every BASELINE config once (stage breakdown), with the info code (GPU box helper)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402
from paper_2412_06551_b200 import _lib  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4a", "cfg4b"]
dev = torch.device("cuda", 0)
for name in names:
    cfg = synth.CONFIGS[name]
    t0 = time.time()
    X = synth.config_matrix(cfg, device=dev)
    plan = rl.Plan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, device=dev)
    res = plan.run(X)
    torch.cuda.synchronize()
    info = res.info()
    _lib.lib().rlhc_stage_timing(1)
    _lib.stage_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = plan.run(X)
    e1.record()
    torch.cuda.synchronize()
    st = _lib.stage_times()
    _lib.lib().rlhc_stage_timing(0)
    Q = res.Q
    orth = torch.linalg.norm(Q.T @ Q - torch.eye(cfg.n, device=dev, dtype=torch.float64)).item()
    resid = (torch.linalg.norm(Q @ res.R - X) / torch.linalg.norm(X)).item()
    print(json.dumps({"cfg": name, "ms": e0.elapsed_time(e1), "info": info, "orth": orth, "resid": resid,
                      "setup_s": round(time.time() - t0, 1),
                      "stages_ms": {k: round(v, 3) for k, v in st.items() if k != "calls"}}), flush=True)
    del X, plan, res, Q
    torch.cuda.empty_cache()
