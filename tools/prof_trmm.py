"""One rlhc_trsm_apply call (mode, m, n from argv) for ncu captures of the pass kernels.

  python tools/prof_trmm.py inv 2097152 256 [gram]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402

mode = rl.RLHC_INV_GEMM if sys.argv[1] == "inv" else rl.RLHC_SUBST
m, n = int(sys.argv[2]), int(sys.argv[3])
gram = len(sys.argv) > 4
dev = torch.device("cuda", 0)
A = torch.randn(m, n, dtype=torch.float64, device=dev)
T = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev)) * 0.1 + 4 * torch.eye(n, dtype=torch.float64, device=dev)
out = torch.empty_like(A)
for _ in range(2):
    rl.trsm_apply(A, T, mode=mode, out=out, want_gram=gram)
torch.cuda.synchronize()
print("ok")
