"""Time rlhc_trsm_apply (SUBST vs INV_GEMM, with / without the Gram) at the pipeline's pass sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
sizes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [(65536, 64), (1 << 20, 128), (262144, 512)]
for (m, n) in sizes:
    A = torch.randn(m, n, dtype=torch.float64, device=dev)
    T = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev)) * 0.1 + 4 * torch.eye(n, dtype=torch.float64, device=dev)
    out = torch.empty_like(A)
    for mode in (rl.RLHC_SUBST, rl.RLHC_INV_GEMM):
        for g in (False, True):
            for _ in range(2):
                rl.trsm_apply(A, T, mode=mode, out=out, want_gram=g)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                rl.trsm_apply(A, T, mode=mode, out=out, want_gram=g)
            e1.record()
            e1.synchronize()
            print(f"m={m} n={n} mode={'inv' if mode else 'subst'} gram={g}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
