"""LU panel-pair split sweep (measurement tool): rlhc_getrf_ts on a seeded m x n matrix under the
(128, 8, 16) contract; prints the time (CUDA events, best of reps) and hashes of the pivots and L,
which must not depend on RLHC_LU_PAIR_SPLIT (the knob is read once per process).

  RLHC_LU_PAIR_SPLIT=60 python tools/lu_split.py 16777216 256 [reps]
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
X = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
piv, U, L11, L, info = rl.getrf_ts(X, cfg=(128, 8, 16), want_L=True)
best = 1e30
for _ in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    piv, U, L11, L, info = rl.getrf_ts(X, cfg=(128, 8, 16), want_L=True)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
h = lambda t: hashlib.sha1(t.contiguous().cpu().numpy().tobytes()).hexdigest()[:12]  # noqa: E731
print(json.dumps({"split": os.environ.get("RLHC_LU_PAIR_SPLIT", "100"), "m": m, "n": n, "ms": round(best, 3),
                  "info": list(info), "piv": h(piv), "U": h(U), "L": h(L)}))
