"""Arrowhead: GPU W = X Y^{-1} and fused G = W^T W vs numpy on the same Y."""
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
X = synth.arrowhead(20000, 50, 1e-25, device=dev)
Xh = X.cpu().numpy()
piv, U, L11, L, info = rl.getrf_ts(X, want_L=True)
Uh, Lh = U.cpu().numpy(), L.cpu().numpy()
Ls = oracle.omega_block(1000, 0, 50, 0, 20000) @ Lh
S = np.linalg.qr(Ls, mode="r")
S = S * (np.sign(np.diag(S)) * np.sign(np.diag(Uh)))[:, None]
Y = S @ Uh
W_np = sl.solve_triangular(Y.T, Xh.T, lower=True).T
W_or = oracle.trsm_right_upper(Xh, Y)
W_gpu, G_gpu, inf = rl.trsm_apply(X, torch.from_numpy(Y).to(dev), want_gram=True)
Wg = W_gpu.cpu().numpy(); Gg = G_gpu.cpu().numpy()
print("info", inf)
print("|W| max", np.abs(W_np).max(), "rows nonzero", int((np.abs(Wg).sum(1) > 0).sum()))
print("W_gpu == W_oracle bitwise:", np.array_equal(Wg, W_or), " rel diff vs numpy W:", np.linalg.norm(Wg - W_np) / np.linalg.norm(W_np))
G1 = Wg.T @ Wg
print("G_gpu vs numpy Gram of W_gpu: rel", np.linalg.norm(Gg - G1) / np.linalg.norm(G1))
print("G_oracle(W_gpu) vs numpy:", np.linalg.norm(oracle.gram(Wg) - G1) / np.linalg.norm(G1))
ev = np.linalg.eigvalsh(G1); print("eig(G) min/max", ev.min(), ev.max())
evg = np.linalg.eigvalsh((Gg + Gg.T) / 2); print("eig(G_gpu) min/max", evg.min(), evg.max())
d = np.abs(Gg - G1); i = np.unravel_index(d.argmax(), d.shape); print("max abs diff at", i, Gg[i], G1[i])
print("W cond", np.linalg.cond(Wg[:50]))
