"""Time the small factorization entry points (HQR, Cholesky) in isolation with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000


g = torch.Generator("cuda").manual_seed(0)
for (s, n) in [(32, 16), (128, 64), (256, 128)]:
    A = torch.randn(s, n, dtype=torch.float64, device="cuda", generator=g)
    G = A.T @ A
    t_h = timeit(lambda: rl.hqr_r(A))
    t_c = timeit(lambda: rl.cholesky(G)) if n <= 150 else float("nan")
    print(f"s={s} n={n}: hqr {t_h:8.1f} us   chol {t_c:8.1f} us   (includes host info readback)")
