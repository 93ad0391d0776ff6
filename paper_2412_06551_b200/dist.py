"""Row-sharded SLHC3 / SSLHC3 over several GPUs.

Rank r holds the global rows [row0, row0 + m_local) of X.  Per call:

* PX = LU: per panel, each rank reduces its leaves and its local tree levels to K
  tournament slots (rlhc_tslu_reduce_to): its rows are K complete subtrees of the global
  tree (K = leaves / the largest power of the arity dividing it, local_slots).  The K slots
  of every rank are all-gathered (global order) and every rank runs the remaining tree levels
  (rlhc_tslu_combine) -> identical pivots everywhere, and the pivots of the single-GPU
  contract: the tree is the global one at every GPU count.  The pivot rows' current values
  are assembled by an all-reduce SUM of per-rank masked copies (rlhc_owned_rows; exact:
  x + 0 + ... + 0 = x), U rows follow (replicated), each rank eliminates its own rows.
* L of the local rows, local sketch partials (Omega columns / CountSketch hashes indexed
  by global row ids) -> all-reduce SUM -> replicated HouseholderQR, Y = S U.
* W = X Y^{-1} with the local Gram partial -> all-reduce -> replicated Cholesky; same for V;
  Q = V J^{-1} stays local; R = J (D Y) replicated.

Only torch.distributed (NCCL over NVLink on GPUs, gloo in CPU tests) moves data here; every
arithmetic step is a call into librlhc.so (CudaBackend).  Tests plug an oracle-backed
backend with the same methods to check this orchestration on CPU.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from ._lib import RLHC_INV_GEMM, RLHC_SUBST, STAGE_CHOL1, STAGE_CHOL2, Info, TsluCfg, check, lib


def kernel_width(panel: int) -> int:
    return 16 if panel <= 16 else 32 if panel <= 32 else 64


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class CudaBackend:
    """Stage calls through the C ABI on the current CUDA stream."""

    def __init__(self, device, cfg: TsluCfg):
        self.dev = torch.device(device)
        self.cfg = cfg
        self.W = kernel_width(cfg.panel)
        self.L = lib()

    def _st(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def _ws(self, nbytes):
        return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=self.dev)

    def _info(self):
        return torch.zeros(2, dtype=torch.int64, device=self.dev)

    # -- tournament
    def new_slot(self, count=1):
        return (torch.full((count, self.W), -1, dtype=torch.int32, device=self.dev),
                torch.zeros(count, dtype=torch.int32, device=self.dev),
                torch.zeros(count, self.W * self.W, dtype=torch.float64, device=self.dev))

    def tslu_reduce(self, src, row0, p0, w, chosen, nslots: int = 1):
        rows = src.shape[0]
        ids, cnt, vals = self.new_slot(nslots)
        ws = self._ws(self.L.rlhc_tslu_local_workspace_size(rows, 0, ctypes.byref(self.cfg)))
        check(self.L.rlhc_tslu_reduce_to(_p(src), src.stride(0), rows, row0, p0, w, _p(chosen),
                                         ctypes.byref(self.cfg), nslots, _p(ids), _p(cnt), _p(vals), _p(ws),
                                         ws.numel(), self._st()))
        return ids, cnt, vals

    def tslu_combine(self, ids, cnt, vals, w):
        nslots = ids.shape[0]
        oi, oc, ov = self.new_slot()
        ws = self._ws(self.L.rlhc_tslu_local_workspace_size(0, nslots, ctypes.byref(self.cfg)))
        check(self.L.rlhc_tslu_combine(_p(ids), _p(cnt), _p(vals), nslots, w, ctypes.byref(self.cfg), _p(oi), _p(oc),
                                       _p(ov), _p(ws), ws.numel(), self._st()))
        return oi, oc, ov

    def owned_rows(self, src, row0, ids, c0, ncols):
        w = ids.numel()
        out = torch.empty(w, ncols, dtype=torch.float64, device=self.dev)
        i32 = ids if ids.dtype == torch.int32 else None
        i64 = ids if ids.dtype == torch.int64 else None
        check(self.L.rlhc_owned_rows(_p(src), src.stride(0), src.shape[0], row0, _p(i32), _p(i64), w, c0, ncols,
                                     _p(out), self._st()))
        return out

    def panel_factor_rows(self, prow, ids, p0, w, n, row0, rows, U, piv, chosen):
        ws = self._ws(self.L.rlhc_tslu_panel_workspace_size(n))
        info = self._info()
        check(self.L.rlhc_tslu_panel_factor_rows(_p(prow), _p(ids), p0, w, n, row0, rows, _p(U), _p(piv), _p(chosen),
                                                 _p(ws), ws.numel(), _p(info), self._st()))
        return info

    # -- left-looking blocks of the warp contract (leaf 128, 16-column panels)
    def warp_contract(self):
        c = self.cfg
        return c.leaf_rows == 128 and 2 <= c.arity <= 8 and c.panel == 16

    def tslw_schur(self, X, L, p0, U):
        check(self.L.rlhc_tslw_schur(_p(X), X.shape[0], X.shape[1], X.stride(0), _p(L), L.stride(0), p0, _p(U),
                                     self._st()))

    def tslw_owned_rows(self, X, L, row0, ids, p0, U):
        n = X.shape[1]
        out = torch.empty(ids.numel(), n - p0, dtype=torch.float64, device=self.dev)
        check(self.L.rlhc_tslw_owned_rows(_p(X), X.stride(0), _p(L), L.stride(0), X.shape[0], row0, _p(ids),
                                          ids.numel(), p0, n, _p(U), _p(out), self._st()))
        return out

    def tslw_finish(self, L, row0, U, piv):
        check(self.L.rlhc_tslw_finish(_p(L), L.stride(0), L.shape[0], row0, L.shape[1], _p(U), _p(piv), self._st()))

    def eliminate(self, src, p0, w, n, U, dst):
        ws = self._ws(self.L.rlhc_tslu_eliminate_workspace_size(n))
        check(self.L.rlhc_tslu_eliminate(_p(src), src.stride(0), src.shape[0], p0, w, n, _p(U), _p(dst),
                                         dst.stride(0), _p(ws), ws.numel(), self._st()))

    def l11(self, Xp, U):
        n = U.shape[0]
        L11 = torch.empty(n, n, dtype=torch.float64, device=self.dev)
        ws = self._ws(self.L.rlhc_lfactor_workspace_size(n, n))
        check(self.L.rlhc_l11(_p(Xp), n, _p(U), _p(L11), _p(ws), ws.numel(), self._st()))
        return L11

    def lfactor(self, X, row0, U, L11, piv, out):
        rows, n = X.shape
        ws = self._ws(self.L.rlhc_lfactor_workspace_size(rows, n))
        check(self.L.rlhc_lfactor(_p(X), rows, n, X.stride(0), row0, _p(U), _p(L11), _p(piv), _p(out), out.stride(0),
                                  _p(ws), ws.numel(), self._st()))
        return out

    # -- sketches and the dense n x n steps
    def sketch_gauss(self, A, row0, s, seed, stream_id):
        rows, n = A.shape
        out = torch.empty(s, n, dtype=torch.float64, device=self.dev)
        ws = self._ws(self.L.rlhc_sketch_gauss_workspace_size(rows, n, s))
        check(self.L.rlhc_sketch_gauss(_p(A), rows, n, A.stride(0), row0, s, seed, stream_id, _p(out), _p(ws),
                                       ws.numel(), self._st()))
        return out

    def sketch_count(self, A, row0, s1, seed):
        rows, n = A.shape
        out = torch.empty(s1, n, dtype=torch.float64, device=self.dev)
        ws = self._ws(self.L.rlhc_sketch_count_workspace_size(rows, n, s1))
        check(self.L.rlhc_sketch_count(_p(A), rows, n, A.stride(0), row0, s1, seed, _p(out), None, None, _p(ws),
                                       ws.numel(), self._st()))
        return out

    def hqr(self, A, sgn_ref):
        s, n = A.shape
        S = torch.empty(n, n, dtype=torch.float64, device=self.dev)
        ws = self._ws(self.L.rlhc_hqr_workspace_size(s, n))
        info = self._info()
        check(self.L.rlhc_hqr_r(_p(A), s, n, A.stride(0), _p(sgn_ref), _p(S), _p(ws), ws.numel(), _p(info),
                                self._st()))
        return S, info

    def trmm(self, A, B):
        n = A.shape[0]
        C = torch.empty(n, n, dtype=torch.float64, device=self.dev)
        check(self.L.rlhc_trmm_upper(_p(A), _p(B), n, _p(C), self._st()))
        return C

    def solve(self, A, T, out, gram: bool, cholqr: bool = False):
        """out = A T^-1 (+ G = out^T out): W by the oracle-order substitution; the CholeskyQR
        passes (cholqr) as on one GPU -- n > 64 the explicit inverse and the triangular product."""
        rows, n = A.shape
        G = torch.zeros(n, n, dtype=torch.float64, device=self.dev) if gram else None
        info = self._info()
        if rows == 0:
            return G, info
        ws = self._ws(self.L.rlhc_trsm_apply_workspace_size(rows, n))
        mode = RLHC_INV_GEMM if cholqr and n > 64 else RLHC_SUBST
        check(self.L.rlhc_trsm_apply(_p(A), rows, n, A.stride(0), _p(T), mode, _p(out), out.stride(0), _p(G),
                                     _p(ws), ws.numel(), _p(info), self._st()))
        return G, info

    def cholesky(self, G, stage):
        n = G.shape[0]
        R = torch.empty(n, n, dtype=torch.float64, device=self.dev)
        ws = self._ws(self.L.rlhc_cholesky_workspace_size(n))
        info = self._info()
        check(self.L.rlhc_cholesky_ws(_p(G), n, _p(R), stage, _p(ws), ws.numel(), _p(info), self._st()))
        return R, info

    def zeros(self, *shape, dtype=torch.float64):
        return torch.zeros(*shape, dtype=dtype, device=self.dev)

    @staticmethod
    def decode(info_t):
        v = info_t.cpu()
        return int(v[0].item() & 0xffffffff), int((v[0].item() >> 32) & 0xffffffff), int(v[1].item())


def local_slots(m_local: int, cfg: TsluCfg) -> int:
    """Slots a rank of m_local rows reduces to: its leaf count divided by the largest power of
    the arity dividing it -- the rank's rows are that many complete subtrees of the global
    tree (rlhc_tslu_local_slots)."""
    k = -(-m_local // cfg.leaf_rows)
    while k % cfg.arity == 0:
        k //= cfg.arity
    return k


def check_shard_contract(m_global: int, m_local: int, world: int, cfg: TsluCfg):
    """Equal shards of whole leaves: each rank's rows are local_slots(m_local) complete
    subtrees of the global tournament tree, so every GPU count runs
    the single-GPU contract's tree and picks its pivots."""
    if cfg.leaf_rows < 1 or cfg.arity < 2 or not 1 <= cfg.panel <= 64:
        raise ValueError("bad tournament contract")
    if m_local * world != m_global:
        raise ValueError("row shards must be equal")
    if world > 1 and m_local % cfg.leaf_rows:
        raise ValueError("m_local must be a multiple of leaf_rows")


class DistPlan:
    """One rank's part of a row-sharded SLHC3 / SSLHC3 call."""

    def __init__(self, algo: str, m_global: int, n: int, s: int = 0, s1: int = 0, s2: int = 0, seed: int = 0,
                 cfg: TsluCfg | None = None, device="cuda", group=None, backend=None):
        self.algo, self.n, self.seed = algo, n, seed
        self.s, self.s1, self.s2 = s, s1, s2
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.m_global = m_global
        self.m_local = m_global // self.world
        self.row0 = self.rank * self.m_local
        self.cfg = cfg if cfg is not None else dist_default_cfg(m_global, n, self.world)
        check_shard_contract(m_global, self.m_local, self.world, self.cfg)
        self.K = local_slots(self.m_local, self.cfg) if self.world > 1 else 1
        self.B = backend if backend is not None else CudaBackend(device, self.cfg)

    # ---- collectives (torch.distributed; no-ops on one rank)
    def _allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _allgather(self, t):
        if self.world == 1:
            return t
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def run(self, X, Q=None):
        """X: this rank's m_local x n rows.  Returns (Q_local, R, piv, info_list)."""
        B, n, cfg = self.B, self.n, self.cfg
        m = X.shape[0]
        assert m == self.m_local and X.shape[1] == n
        Q = Q if Q is not None else B.zeros(m, n)
        infos = []
        # ---------------- PX = LU (tournament over panels), P:279 / P:293
        U = B.zeros(n, n)
        piv = B.zeros(n, dtype=torch.int64)
        chosen = B.zeros(m, dtype=torch.uint8)
        if getattr(B, "warp_contract", lambda: False)() and n > 16:
            # left-looking panels (the single-process pipeline's arithmetic): this rank's Schur
            # complement of the panel into Q, the local tournament, the gathered top levels, the
            # winners' current rows from their owners (all-reduced), their elimination -> U rows
            for p0 in range(0, n, cfg.panel):
                w = min(cfg.panel, n - p0)
                B.tslw_schur(X, Q, p0, U)
                ids, cnt, vals = B.tslu_reduce(Q, self.row0, p0, w, chosen if p0 > 0 else None, self.K)
                if self.world > 1:
                    ids, cnt, vals = B.tslu_combine(self._allgather(ids), self._allgather(cnt),
                                                    self._allgather(vals), w)
                root = ids[0, :w].contiguous()
                prow = self._allreduce(B.tslw_owned_rows(X, Q, self.row0, root, p0, U))
                infos.append(B.panel_factor_rows(prow, root, p0, w, n, self.row0, m, U, piv, chosen))
            B.tslw_finish(Q, self.row0, U, piv)
            L = Q
        else:
            L = None
        for p0 in (range(0, n, cfg.panel) if L is None else ()):
            w = min(cfg.panel, n - p0)
            src = X if p0 == 0 else Q
            ids, cnt, vals = B.tslu_reduce(src, self.row0, p0, w, chosen if p0 > 0 else None, self.K)
            if self.world > 1:
                ids, cnt, vals = B.tslu_combine(self._allgather(ids), self._allgather(cnt), self._allgather(vals), w)
            root = ids[0, :w].contiguous()
            prow = self._allreduce(B.owned_rows(src, self.row0, root, p0, n - p0))
            infos.append(B.panel_factor_rows(prow, root, p0, w, n, self.row0, m, U, piv, chosen))
            if p0 + w < n:
                B.eliminate(src, p0, w, n, U, Q)
        if L is None:
            Xp = self._allreduce(B.owned_rows(X, self.row0, piv, 0, n))
            L11 = B.l11(Xp, U)
            L = B.lfactor(X, self.row0, U, L11, piv, Q)
        # ---------------- sketch of L (P:280 / P:294), all-reduced partials
        if self.algo == "slhc3":
            Ls = self._allreduce(B.sketch_gauss(L, self.row0, self.s, self.seed, 0))
        else:
            Lt = self._allreduce(B.sketch_count(L, self.row0, self.s1, self.seed))
            Ls = B.sketch_gauss(Lt, 0, self.s2, self.seed, 1)
        S, info = B.hqr(Ls, U)
        infos.append(info)
        Y = B.trmm(S, U)
        # ---------------- W = X Y^{-1} (+G1), CholeskyQR2, R = J (D Y)
        G1, info = B.solve(X, Y, Q, gram=True)
        infos.append(info)
        D, info = B.cholesky(self._allreduce(G1), STAGE_CHOL1)
        infos.append(info)
        G2, info = B.solve(Q, D, Q, gram=True, cholqr=True)
        infos.append(info)
        J, info = B.cholesky(self._allreduce(G2), STAGE_CHOL2)
        infos.append(info)
        _, info = B.solve(Q, J, Q, gram=False, cholqr=True)
        infos.append(info)
        R = B.trmm(J, B.trmm(D, Y))
        return Q, R, piv, infos

    def first_error(self, infos):
        for t in infos:
            code = self.B.decode(t)
            if code[0] != 0:
                return code
        return (0, 0, 0)


class _DistResult:
    def __init__(self, plan, Q, R, piv, infos):
        self.plan, self.Q, self.R, self.piv, self.infos = plan, Q, R, piv, infos

    def info(self):
        return self.plan.first_error(self.infos)


class BenchRunner:
    """bench.py's N > 1 step: this rank's rows of the weak-scaled workload."""

    def __init__(self, plan: DistPlan):
        self.plan = plan
        self.Q = plan.B.zeros(plan.m_local, plan.n)

    def run(self, X):
        Q, R, piv, infos = self.plan.run(X, self.Q)
        return _DistResult(self.plan, Q, R, piv, infos)


def setup_bench(cfg, rank: int, world: int, device, strong: bool = True, use_c: bool = True, contract=None):
    """bench.py's N-GPU workload.  Strong scaling (bench.py's default at N > 1): the job factors
    cfg's m x n X, each rank holds m / world rows.  Weak scaling (--weak): every rank holds cfg.m
    rows of a (world * cfg.m) x n X.  Either way the contract is the single-GPU default
    (dist_default_cfg: 128-row leaves, 8-ary nodes, 16-column panels): a rank's equal shard of
    whole leaves is a union of complete subtrees of the global tournament tree,
    so the pivots equal a single-GPU run on the whole X."""
    import synth
    m_global = cfg.m if strong else cfg.m * world
    m_local = m_global // world
    X = synth.baseline_matrix(m_global, cfg.n, cfg.kappa_exp, cfg.seed, cfg.colscale, device=device,
                              row0=rank * m_local, rows=m_local)
    tc = TsluCfg(*contract) if contract is not None else dist_default_cfg(m_global, cfg.n, world)
    if use_c:  # the C orchestration (rlhc_*_dist) over an NCCL communicator of its own
        plan = CDistPlan(cfg.algo, m_global, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, cfg=tc,
                         device=device, comm=NcclComm())
        return X, plan
    plan = DistPlan(cfg.algo, m_global, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, cfg=tc, device=device)
    return X, BenchRunner(plan)


def dist_default_cfg(m_global: int, n: int, world: int) -> TsluCfg:
    """The single-GPU default contract (rlhc_default_tslu_cfg: 128-row leaves, 8-ary nodes,
    16-column panels) at every GPU count: equal shards of whole leaves are unions of complete
    subtrees of its global tree, so the pivots equal the single-GPU run's."""
    c = TsluCfg()
    lib().rlhc_default_tslu_cfg(m_global, n, ctypes.byref(c))
    return c


# ---------------------------------------------------------------- C orchestration over NCCL
class NcclComm:
    """An NCCL communicator for the C entry points (rlhc_comm_init).  Rank 0's unique id is
    distributed with torch.distributed (plumbing only); nranks == 1 needs no process group."""

    def __init__(self, group=None):
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            check(lib().rlhc_comm_unique_id(uid))
        if self.world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            ctypes.memmove(uid, box[0], 128)
        self.handle = ctypes.c_void_p()
        check(lib().rlhc_comm_init(ctypes.byref(self.handle), self.world, self.rank, uid))

    def close(self):
        if self.handle:
            lib().rlhc_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CDistPlan:
    """One rank's row-sharded SLHC3 / SSLHC3 through rlhc_slhc3_dist / rlhc_sslhc3_dist: the
    whole call (tournament, sketches, factorizations, NCCL collectives) in C on the current
    stream.  Same contract and shard rules as DistPlan."""

    def __init__(self, algo: str, m_global: int, n: int, s: int = 0, s1: int = 0, s2: int = 0, seed: int = 0,
                 cfg: TsluCfg | None = None, device="cuda", comm: NcclComm | None = None):
        self.algo, self.n, self.seed, self.s, self.s1, self.s2 = algo, n, seed, s, s1, s2
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.m_global, self.m_local = m_global, m_global // self.world
        self.row0 = self.rank * self.m_local
        self.cfg = cfg if cfg is not None else dist_default_cfg(m_global, n, self.world)
        check_shard_contract(m_global, self.m_local, self.world, self.cfg)
        self.dev = torch.device(device)
        aid = 0 if algo == "slhc3" else 1
        nbytes = lib().rlhc_dist_workspace_size(aid, self.m_local, n, s if aid == 0 else s1, s2, ctypes.byref(self.cfg),
                                                self.world)
        if nbytes == 0:
            raise ValueError("unsupported sizes for the distributed entry point")
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.dev)
        off = (-self.ws.data_ptr()) % 256
        self.ws_ptr, self.ws_bytes = self.ws.data_ptr() + off, nbytes
        self.Q = torch.empty(self.m_local, n, dtype=torch.float64, device=self.dev)
        self.R = torch.empty(n, n, dtype=torch.float64, device=self.dev)
        self.piv = torch.empty(n, dtype=torch.int64, device=self.dev)
        self.info_t = torch.zeros(2, dtype=torch.int64, device=self.dev)

    def run(self, X):
        assert X.shape == (self.m_local, self.n) and X.dtype == torch.float64
        st = ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        h = self.comm.handle if self.comm is not None else None
        common = (ctypes.c_void_p(X.data_ptr()), self.m_local, self.n, X.stride(0), self.row0, self.m_global)
        tail = (ctypes.c_uint64(self.seed), ctypes.byref(self.cfg), ctypes.c_void_p(self.Q.data_ptr()),
                self.Q.stride(0), ctypes.c_void_p(self.R.data_ptr()), ctypes.c_void_p(self.piv.data_ptr()),
                ctypes.c_void_p(self.ws_ptr), self.ws_bytes, ctypes.c_void_p(self.info_t.data_ptr()), h, st)
        if self.algo == "slhc3":
            check(lib().rlhc_slhc3_dist(*common, self.s, *tail))
        else:
            check(lib().rlhc_sslhc3_dist(*common, self.s1, self.s2, *tail))
        return _CResult(self)


class _CResult:
    def __init__(self, plan):
        self.plan, self.Q, self.R, self.piv = plan, plan.Q, plan.R, plan.piv

    def info(self):
        v = self.plan.info_t.cpu()
        code = int(v[0] & 0xffffffff)
        stage = int((v[0] >> 32) & 0xffffffff)
        return code, stage, int(v[1])
