"""Oracle-backed stage backend for paper_2412_06551_b200.dist.DistPlan (CPU tests only).

Implements the same methods as dist.CudaBackend with the CPU oracle's arithmetic on CPU
torch tensors, so the row-sharded orchestration (tournament slots, all-gathers,
all-reduces, replicated small factorizations) can be exercised with the gloo backend and
world size 2 in a GPU-less container.  Test infrastructure: never used by the product.
"""
import numpy as np
import torch

import oracle


class OracleBackend:
    def __init__(self, cfg):
        self.cfg = cfg
        p = cfg.panel
        self.W = 16 if p <= 16 else 32 if p <= 32 else 64

    # ---------------------------------------------------------------- helpers
    def zeros(self, *shape, dtype=torch.float64):
        return torch.zeros(*shape, dtype=dtype)

    def _info(self, code=0, stage=0, index=0):
        return torch.tensor([(stage << 32) | code, index], dtype=torch.int64)

    @staticmethod
    def decode(info_t):
        v = info_t.cpu()
        return int(v[0].item() & 0xffffffff), int((v[0].item() >> 32) & 0xffffffff), int(v[1].item())

    def _slot(self, ids, vals, w):
        W = self.W
        si = torch.full((1, W), -1, dtype=torch.int32)
        sc = torch.zeros(1, dtype=torch.int32)
        sv = torch.zeros(1, W * W, dtype=torch.float64)
        k = len(ids)
        si[0, :k] = torch.from_numpy(np.asarray(ids, np.int32))
        sc[0] = k
        if k:
            v = np.zeros((W, W))
            v[:k, :w] = vals
            sv[0] = torch.from_numpy(v.reshape(-1))
        return si, sc, sv

    def _select(self, cand_ids, cand_vals, w):
        if len(cand_ids) == 0:
            return np.zeros(0, np.int64), np.zeros((0, w))
        win = oracle.select(cand_vals, cand_ids, w)
        pos = {int(i): r for r, i in enumerate(cand_ids)}
        return win, np.stack([cand_vals[pos[int(i)]] for i in win])

    def _tree(self, slots, w, target=None):
        """Tree levels over `slots` down to one slot (returned), or down to `target` slots
        (returned as a list) when given."""
        while len(slots) > (target or 1):
            nxt = []
            for c0 in range(0, len(slots), self.cfg.arity):
                grp = slots[c0:c0 + self.cfg.arity]
                ids = np.concatenate([g[0] for g in grp])
                vals = np.concatenate([g[1] for g in grp]) if len(ids) else np.zeros((0, w))
                nxt.append(self._select(ids, vals, w))
            slots = nxt
        return slots if target else slots[0]

    # ---------------------------------------------------------------- tournament
    def tslu_reduce(self, src, row0, p0, w, chosen, nslots=1):
        A = src.numpy()
        rows = A.shape[0]
        ch = chosen.numpy() if chosen is not None else np.zeros(rows, np.uint8)
        b = self.cfg.leaf_rows
        slots = []
        for l0 in range(0, rows, b):
            loc = [i for i in range(l0, min(rows, l0 + b)) if not ch[i]]
            ids = np.array([row0 + i for i in loc], np.int64)
            vals = A[loc, p0:p0 + w].copy() if loc else np.zeros((0, w))
            slots.append(self._select(ids, vals, w))
        slots = self._tree(slots, w, nslots)
        out = [self._slot(i, v, w) for i, v in slots]
        return tuple(torch.cat([o[j] for o in out]) for j in range(3))

    def tslu_combine(self, ids, cnt, vals, w):
        W = self.W
        slots = []
        for g in range(ids.shape[0]):
            k = int(cnt[g])
            slots.append((ids[g, :k].numpy().astype(np.int64), vals[g].numpy().reshape(W, W)[:k, :w].copy()))
        ids_, vals_ = self._tree(slots, w)
        return self._slot(ids_, vals_, w)

    def owned_rows(self, src, row0, ids, c0, ncols):
        A = src.numpy()
        out = np.zeros((ids.numel(), ncols))
        for t, g in enumerate(ids.numpy().astype(np.int64)):
            lr = g - row0
            if 0 <= lr < A.shape[0]:
                out[t] = A[lr, c0:c0 + ncols]
        return torch.from_numpy(out)

    def panel_factor_rows(self, prow, ids, p0, w, n, row0, rows, U, piv, chosen):
        P = oracle.panel_rows(prow.numpy())
        Un = U.numpy()
        for t in range(w):
            Un[p0 + t, p0 + t:] = P[t, t:]
            g = int(ids[t])
            piv[p0 + t] = g
            if 0 <= g - row0 < rows:
                chosen[g - row0] = 1
        for t in range(w):
            if P[t, t] == 0.0:
                return self._info(oracle.ERANKDEF, oracle.ST_LU, p0 + t)
        return self._info()

    def eliminate(self, src, p0, w, n, U, dst):
        # every row is eliminated (as on the GPU): rows already chosen as pivots are never read again
        if dst.data_ptr() != src.data_ptr():
            dst.copy_(src)
        oracle.eliminate_rows(dst.numpy(), p0, w, U.numpy(), np.zeros(dst.shape[0], np.uint8))

    def l11(self, Xp, U):
        n = U.shape[0]
        L = oracle.lfactor_rows(Xp.numpy(), -(1 << 40), np.full(n, -1, np.int64), U.numpy(), np.zeros((n, n)))
        L = np.tril(L, -1) + np.eye(n)
        return torch.from_numpy(L)

    def lfactor(self, X, row0, U, L11, piv, out):
        out.copy_(torch.from_numpy(oracle.lfactor_rows(X.numpy(), row0, piv.numpy(), U.numpy(), L11.numpy())))
        return out

    # ---------------------------------------------------------------- dense
    def sketch_gauss(self, A, row0, s, seed, stream_id):
        return torch.from_numpy(oracle.sketch_gauss(A.numpy(), s, seed, stream_id, row0=row0))

    def sketch_count(self, A, row0, s1, seed):
        b, sg = oracle.cs_hash(seed, row0, A.shape[0], s1)
        return torch.from_numpy(oracle.cs_apply(A.numpy(), b, sg, s1))

    def hqr(self, A, sgn_ref):
        S = oracle.hqr_r(A.numpy())
        d = np.diag(sgn_ref.numpy())
        flip = (np.diag(S) < 0) != (d < 0)
        S[flip] = -S[flip]
        return torch.from_numpy(S), self._info()

    def trmm(self, A, B):
        return torch.from_numpy(oracle.trmm_uu(A.numpy(), B.numpy()))

    def solve(self, A, T, out, gram, cholqr=False):
        res = oracle.trsm_right_upper(A.numpy(), T.numpy())
        out.copy_(torch.from_numpy(res))
        G = torch.from_numpy(oracle.gram(res)) if gram else None
        return G, self._info()

    def cholesky(self, G, stage):
        try:
            return torch.from_numpy(oracle.chol(G.numpy(), stage)), self._info()
        except oracle.OracleError as e:
            n = G.shape[0]
            return torch.zeros(n, n, dtype=torch.float64), self._info(e.code, e.stage, e.index)
