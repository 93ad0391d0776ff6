"""GPU vs oracle on the arrowhead: info codes and the LU outputs bit for bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

beta = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-25
dev = torch.device("cuda", 0)
X = synth.arrowhead(20000, 50, beta, device=dev)
Xh = X.cpu().numpy()
piv, U, L11, L, info = rl.getrf_ts(X, want_L=True)
opiv, oU, oL11, oL = oracle.tslu(Xh, 128, 8, 16, want_L=True)
print("getrf info", info)
print("piv equal", np.array_equal(piv.cpu().numpy(), opiv))
for nm, a, b in (("U", U, oU), ("L11", L11, oL11), ("L", L, oL)):
    a = a.cpu().numpy()
    d = np.argwhere(~((a == b) | (np.isnan(a) & np.isnan(b))))
    print(nm, "mismatches", len(d), d[:5].tolist(), [(a[tuple(i)], b[tuple(i)]) for i in d[:3]])
for seed in range(1000, 1004):
    r = rl.slhc3(X, 50, seed=seed)
    ro = oracle.slhc3(Xh, 50, seed, 128, 8, 16, raise_on_error=False)
    print("seed", seed, "gpu", r.info(), "oracle", ro.info)
    ro2 = oracle.slhc3(Xh, 50, seed, 128, 8, 16, stages=True, raise_on_error=False)
    print("  oracle stage arrays", {k: float(np.abs(v).max()) for k, v in ro2[3].items()} if len(ro2) > 3 else None)
