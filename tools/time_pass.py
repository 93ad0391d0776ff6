"""Time one streaming pass at a pipeline size under the current measurement knobs (env), and
print a bit-level checksum of its output so that variants can be compared bit for bit.

  python tools/time_pass.py subst|inv|gram M N [reps]

subst: W = A T^-1 by the oracle-order substitution (rlhc_trsm_apply RLHC_SUBST, no Gram);
inv: the same through the explicit inverse + DMMA product (RLHC_INV_GEMM);
gram: G = A^T A (rlhc_gram).  A is seeded N(0,1), T = 0.1 triu(N(0,1)) + 4 I.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402

what, m, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
A = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
T = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)) * 0.1 + \
    4 * torch.eye(n, dtype=torch.float64, device=dev)
out = torch.empty_like(A) if what != "gram" else None


def run():
    if what == "gram":
        return rl.gram(A)
    rl.trsm_apply(A, T, mode=rl.RLHC_SUBST if what == "subst" else rl.RLHC_INV_GEMM, out=out)
    return out


for _ in range(2):
    res = run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
res = run()
torch.cuda.synchronize()
bits = res.contiguous().view(torch.int64)
chk = int(bits.remainder(1000003).sum().item()) * 7 + int(bits[::3].remainder(999983).sum().item())
knobs = {k: v for k, v in os.environ.items() if k.startswith("RLHC_")}
ts.sort()
print(f"{what} m={m} n={n} knobs={knobs} median_ms={ts[len(ts) // 2]:.3f} min_ms={ts[0]:.3f} checksum={chk}",
      flush=True)
