"""Debug helper: getrf_ts on a rank-deficient multi-panel matrix."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_06551_b200 as rl  # noqa: E402

m, n, col = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
X = synth.baseline_matrix(m, n, 12, 8, device="cuda")
X[:, col] = 0.0
piv, U, L11, L, info = rl.getrf_ts(X, cfg=(256, 2, 64))
torch.cuda.synchronize()
print(sys.argv[1:], "info", info, "U diag finite", bool(torch.isfinite(torch.diagonal(U)).all()), flush=True)
