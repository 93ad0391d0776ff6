"""Debug helper: DistPlan (Python orchestration) on a rank-deficient 2-panel input."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_06551_b200._lib import TsluCfg  # noqa: E402
from paper_2412_06551_b200.dist import DistPlan  # noqa: E402

m, n = 16384, 100
X = synth.baseline_matrix(m, n, 12, 8, device="cuda")
X[:, 5] = 0.0
plan = DistPlan("sslhc3", m, n, s1=800, s2=200, seed=3, cfg=TsluCfg(256, 2, 64), device="cuda")
Q, R, piv, infos = plan.run(X)
torch.cuda.synchronize()
print("py info", plan.first_error(infos), piv[:8].tolist(), flush=True)
