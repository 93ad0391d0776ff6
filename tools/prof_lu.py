"""rlhc_getrf_ts calls (m, n from argv; default contract) for ncu captures of the LU kernels.

  python tools/prof_lu.py 4194304 256 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda", 0)
X = torch.randn(m, n, dtype=torch.float64, device=dev)
for _ in range(reps):
    rl.getrf_ts(X, cfg=(128, 8, 16), want_L=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rl.getrf_ts(X, cfg=(128, 8, 16), want_L=True)
e1.record()
e1.synchronize()
print(f"getrf_ts m={m} n={n}: {e0.elapsed_time(e1):.3f} ms")
