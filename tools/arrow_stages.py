"""Which stage loses the arrowhead at beta = 1e-25: GPU stage entry points
mixed with numpy/LAPACK stages on the same L (bit-exact between GPU and oracle)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
X = synth.arrowhead(20000, 50, float(sys.argv[1]) if len(sys.argv) > 1 else 1e-25, device=dev)
Xh = X.cpu().numpy()
piv, U, L11, L, info = rl.getrf_ts(X, want_L=True)
Uh, Lh = U.cpu().numpy(), L.cpu().numpy()
g = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731


def ok_np(G):
    try:
        np.linalg.cholesky(G)
        return True
    except np.linalg.LinAlgError:
        return False


res = collections.defaultdict(collections.Counter)
for seed in range(1000, 1040):
    Ls_np = oracle.omega_block(seed, 0, 50, 0, 20000) @ Lh
    Ls_gpu = rl.sketch_gauss(L, 50, seed, 0).cpu().numpy()
    for lsn, Ls in (("Ls_np", Ls_np), ("Ls_gpu", Ls_gpu)):
        S_np = np.linalg.qr(Ls, mode="r")
        S_np = S_np * (np.sign(np.diag(S_np)) * np.sign(np.diag(Uh)))[:, None]
        S_gpu = rl.hqr_r(g(Ls), sgn_ref=U)[0].cpu().numpy()
        for sn, S in (("S_np", S_np), ("S_gpu", S_gpu)):
            Y = S @ Uh
            W_np = sl.solve_triangular(Y.T, Xh.T, lower=True).T
            W_gpu, G_gpu, inf = rl.trsm_apply(X, g(Y), want_gram=True)
            G_np = W_np.T @ W_np
            res[f"{lsn}+{sn}+np"]["ok" if ok_np(G_np) else "bd"] += 1
            if G_gpu is not None:
                res[f"{lsn}+{sn}+gpuW,G"]["ok" if ok_np(G_gpu.cpu().numpy()) else "bd"] += 1
                _, ci = rl.cholesky(G_gpu)
                res[f"{lsn}+{sn}+gpuW,G+gpuchol"]["ok" if ci[0] == 0 else "bd"] += 1
for k, v in sorted(res.items()):
    print(k, dict(v))
