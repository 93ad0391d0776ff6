"""B200-native hot path of randomized LU-Householder CholeskyQR (arXiv 2412.06551).

Thin torch-facing binding of the C ABI in include/rlhc.h: every function below only
allocates device tensors (outputs + workspace) and passes raw pointers and the
current CUDA stream to librlhc.so, whose sm_100a kernels do all the arithmetic.
There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (RLHC_INV_GEMM, RLHC_SLHC3, RLHC_SSLHC3, RLHC_SUBST, STAGE_CHOL1, STAGE_CHOL2, Info, RlhcError,
                   TsluCfg, check, lib)

__all__ = ["slhc3", "sslhc3", "cholqr2", "scholqr3", "luc2", "rhc", "MethodPlan", "getrf_ts", "sketch_gauss", "sketch_count", "gram", "trsm_apply", "hqr_r", "cholesky",
           "default_cfg", "Plan", "RlhcError", "RLHC_SUBST", "RLHC_INV_GEMM", "STAGE_CHOL1", "STAGE_CHOL2"]


def _p(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=torch.float64):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    if t.dim() == 2 and t.stride(1) != 1:
        raise ValueError(f"{name} must be row-major (stride(1) == 1)")


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def default_cfg(m: int, n: int) -> TsluCfg:
    c = TsluCfg()
    lib().rlhc_default_tslu_cfg(m, n, ctypes.byref(c))
    return c


def _cfg(cfg, m, n) -> TsluCfg:
    if cfg is None:
        return default_cfg(m, n)
    if isinstance(cfg, TsluCfg):
        return cfg
    leaf_rows, arity, panel = cfg
    return TsluCfg(leaf_rows, arity, panel)


@dataclass
class Result:
    Q: torch.Tensor
    R: torch.Tensor
    piv: torch.Tensor
    info_dev: torch.Tensor

    def info(self):
        """(code, stage, index) read back from the device (synchronises)."""
        v = self.info_dev.cpu()
        code = int(v[0].item() & 0xffffffff)
        stage = int((v[0].item() >> 32) & 0xffffffff)
        return code, stage, int(v[1].item())


def _new_info(device) -> torch.Tensor:
    # rlhc_info_t = {int32 code; int32 stage; int64 index} == two int64 words (little endian)
    return torch.zeros(2, dtype=torch.int64, device=device)


class Plan:
    """Reusable SLHC3 / SSLHC3 call: workspace, Q, R, piv and info allocated once."""

    def __init__(self, algo: str, m: int, n: int, s: int = 0, s1: int = 0, s2: int = 0, seed: int = 0, cfg=None,
                 device="cuda"):
        self.algo = RLHC_SLHC3 if algo == "slhc3" else RLHC_SSLHC3
        self.m, self.n, self.seed = m, n, seed
        self.a, self.b = (s, 0) if self.algo == RLHC_SLHC3 else (s1, s2)
        self.device = torch.device(device)
        self.cfg = _cfg(cfg, m, n)
        nbytes = lib().rlhc_workspace_size(self.algo, m, n, self.a, self.b, ctypes.byref(self.cfg))
        if nbytes == 0:
            raise RlhcError(_lib.RLHC_EINVAL, "invalid sizes / configuration")
        self.ws = _ws(nbytes, self.device)
        self.Q = torch.empty(m, n, dtype=torch.float64, device=self.device)
        self.R = torch.empty(n, n, dtype=torch.float64, device=self.device)
        self.piv = torch.empty(n, dtype=torch.int64, device=self.device)
        self.info_dev = _new_info(self.device)

    def run(self, X: torch.Tensor) -> Result:
        _need(X, "X")
        m, n = X.shape
        assert (m, n) == (self.m, self.n)
        L = lib()
        args = (_p(X), m, n, X.stride(0))
        tail = (self.seed, ctypes.byref(self.cfg), _p(self.Q), n, _p(self.R), _p(self.piv), _p(self.ws),
                self.ws.numel(), _p(self.info_dev), _stream(self.device))
        if self.algo == RLHC_SLHC3:
            rc = L.rlhc_slhc3(*args, self.a, *tail)
        else:
            rc = L.rlhc_sslhc3(*args, self.a, self.b, *tail)
        check(rc)
        return Result(self.Q, self.R, self.piv, self.info_dev)

    def capture(self, X: torch.Tensor) -> None:
        """Record run(X) as a CUDA graph (rlhc_graph_*); replay() then
        reruns the whole call on X's current contents with one graph launch."""
        self.run(X)  # first launches (module loading) outside the capture
        torch.cuda.synchronize(self.device)
        side = torch.cuda.Stream(device=self.device)
        with torch.cuda.stream(side):
            st = _stream(self.device)
            check(lib().rlhc_graph_begin(st))
            g = ctypes.c_void_p()
            try:
                self.run(X)
            finally:
                rc = lib().rlhc_graph_end(st, ctypes.byref(g))
            check(rc)
        self.release_graph()
        self._graph = g

    def replay(self) -> Result:
        check(lib().rlhc_graph_launch(self._graph, _stream(self.device)))
        return Result(self.Q, self.R, self.piv, self.info_dev)

    def release_graph(self) -> None:
        g = getattr(self, "_graph", None)
        if g is not None and g.value:
            lib().rlhc_graph_destroy(g)
        self._graph = None

    def __del__(self):
        try:
            self.release_graph()
        except Exception:
            pass


def slhc3(X: torch.Tensor, s: int, seed: int = 0, cfg=None) -> Result:
    """SLHC3 (PAPER.md alg:SLHC3) on a CUDA fp64 row-major X (m x n)."""
    m, n = X.shape
    return Plan("slhc3", m, n, s=s, seed=seed, cfg=cfg, device=X.device).run(X)


def sslhc3(X: torch.Tensor, s1: int, s2: int, seed: int = 0, cfg=None) -> Result:
    """SSLHC3 (PAPER.md alg:SSLHC3) on a CUDA fp64 row-major X (m x n)."""
    m, n = X.shape
    return Plan("sslhc3", m, n, s1=s1, s2=s2, seed=seed, cfg=cfg, device=X.device).run(X)


class HostPipeline:
    """Host-buffer pipeline (rlhc_host_pipeline): independent SLHC3 / SSLHC3 problems of one
    shape from host X to host Q, R, piv, info, with the host->device copy of the next problem
    and the device->host copy of the previous one overlapping the current computation."""

    def __init__(self, algo: str, m: int, n: int, s: int = 0, s1: int = 0, s2: int = 0, cfg=None, device="cuda"):
        self.algo = RLHC_SLHC3 if algo == "slhc3" else RLHC_SSLHC3
        self.m, self.n = m, n
        self.a, self.b = (s, 0) if self.algo == RLHC_SLHC3 else (s1, s2)
        self.device = torch.device(device)
        self.cfg = _cfg(cfg, m, n)
        nbytes = lib().rlhc_host_pipeline_workspace_size(self.algo, m, n, self.a, self.b, ctypes.byref(self.cfg))
        if nbytes == 0:
            raise RlhcError(_lib.RLHC_EINVAL, "invalid sizes / configuration")
        self.ws = _ws(nbytes, self.device)

    def run(self, Xs, seeds, Qs, Rs, pivs=None) -> torch.Tensor:
        """Enqueue len(Xs) problems; Xs, Qs, Rs (and pivs) are host tensors (pinned for overlap).
        Returns the infos as a pinned (count, 2) int64 host tensor, valid after
        torch.cuda.synchronize(): use infos() for (code, stage, index) tuples."""
        cnt = len(Xs)
        if len(seeds) != cnt or len(Qs) != cnt or len(Rs) != cnt or (pivs is not None and len(pivs) != cnt):
            raise RlhcError(_lib.RLHC_EINVAL, "Xs, seeds, Qs, Rs (and pivs) must have the same length")
        for t in list(Xs) + list(Qs) + list(Rs):
            if t.device.type != "cpu" or t.dtype != torch.float64 or not t.is_contiguous():
                raise RlhcError(_lib.RLHC_EINVAL, "host buffers must be contiguous float64 CPU tensors")
        ptrs = lambda ts: (ctypes.c_void_p * cnt)(*[t.data_ptr() for t in ts])  # noqa: E731
        xs, qs, rs = ptrs(Xs), ptrs(Qs), ptrs(Rs)
        ps = ptrs(pivs) if pivs is not None else None
        sd = (ctypes.c_uint64 * cnt)(*seeds)
        self._keep = (xs, qs, rs, ps, sd)  # alive until the copies ran
        self.info = torch.zeros(max(cnt, 1), 2, dtype=torch.int64).pin_memory()  # rlhc_info_t[cnt]
        check(lib().rlhc_host_pipeline(self.algo, cnt, xs, self.m, self.n, self.a, self.b, sd, ctypes.byref(self.cfg),
                                       qs, rs, ps, self.info.data_ptr(), _p(self.ws), self.ws.numel(),
                                       _stream(self.device)))
        return self.info

    def infos(self) -> list:
        """(code, stage, index) per problem of the last run (after synchronising)."""
        out = []
        for w0, idx in self.info.tolist():
            out.append((w0 & 0xFFFFFFFF, (w0 >> 32) & 0xFFFFFFFF, idx))
        return out


class MethodPlan:
    """Reusable call of one of the paper's comparison algorithms:
    'cholqr2', 'scholqr3', 'luc2' (tournament contract cfg) or 'rhc' (sketch sizes s1, s2)."""

    IDS = {"cholqr2": _lib.RLHC_CHOLQR2, "scholqr3": _lib.RLHC_SCHOLQR3, "luc2": _lib.RLHC_LUC2, "rhc": _lib.RLHC_RHC}

    def __init__(self, method: str, m: int, n: int, s1: int = 0, s2: int = 0, seed: int = 0, cfg=None,
                 device="cuda"):
        self.method, self.mid = method, self.IDS[method]
        self.m, self.n, self.s1, self.s2, self.seed = m, n, s1, s2, seed
        self.device = torch.device(device)
        self.cfg = _cfg(cfg, m, n)
        nbytes = lib().rlhc_method_workspace_size(self.mid, m, n, s1, s2, ctypes.byref(self.cfg))
        if nbytes == 0:
            raise RlhcError(_lib.RLHC_EINVAL, "invalid sizes / configuration")
        self.ws = _ws(nbytes, self.device)
        self.Q = torch.empty(m, n, dtype=torch.float64, device=self.device)
        self.R = torch.empty(n, n, dtype=torch.float64, device=self.device)
        self.piv = torch.empty(n, dtype=torch.int64, device=self.device)
        self.info_dev = _new_info(self.device)

    def run(self, X: torch.Tensor) -> Result:
        _need(X, "X")
        m, n = X.shape
        assert (m, n) == (self.m, self.n)
        L = lib()
        head = (_p(X), m, n, X.stride(0))
        out = (_p(self.Q), n, _p(self.R))
        tail = (_p(self.ws), self.ws.numel(), _p(self.info_dev), _stream(self.device))
        if self.method == "cholqr2":
            rc = L.rlhc_cholqr2(*head, *out, *tail)
        elif self.method == "scholqr3":
            rc = L.rlhc_scholqr3(*head, *out, *tail)
        elif self.method == "luc2":
            rc = L.rlhc_luc2(*head, ctypes.byref(self.cfg), *out, _p(self.piv), *tail)
        else:
            rc = L.rlhc_rhc(*head, self.s1, self.s2, ctypes.c_uint64(self.seed), *out, *tail)
        check(rc)
        return Result(self.Q, self.R, self.piv, self.info_dev)


def cholqr2(X: torch.Tensor) -> Result:
    """CholeskyQR2 (alg:cholqr2)."""
    return MethodPlan("cholqr2", *X.shape, device=X.device).run(X)


def scholqr3(X: torch.Tensor) -> Result:
    """SCholeskyQR3 (alg:Shifted3; shift P:984)."""
    return MethodPlan("scholqr3", *X.shape, device=X.device).run(X)


def luc2(X: torch.Tensor, cfg=None) -> Result:
    """LU-CholeskyQR2 (alg:LU2)."""
    return MethodPlan("luc2", *X.shape, cfg=cfg, device=X.device).run(X)


def rhc(X: torch.Tensor, s1: int, s2: int, seed: int = 0) -> Result:
    """Rand.Householder-Cholesky (alg:Rand2)."""
    return MethodPlan("rhc", *X.shape, s1=s1, s2=s2, seed=seed, device=X.device).run(X)


def getrf_ts(X: torch.Tensor, cfg=None, want_L: bool = False):
    """PX = LU under the tournament contract: (piv, U, L11, L or None, info)."""
    _need(X, "X")
    m, n = X.shape
    dev = X.device
    c = _cfg(cfg, m, n)
    ws = _ws(lib().rlhc_getrf_ts_workspace_size(m, n, ctypes.byref(c)), dev)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    U = torch.empty(n, n, dtype=torch.float64, device=dev)
    L11 = torch.empty(n, n, dtype=torch.float64, device=dev)
    L = torch.empty(m, n, dtype=torch.float64, device=dev) if want_L else None
    info = _new_info(dev)
    check(lib().rlhc_getrf_ts(_p(X), m, n, X.stride(0), 0, ctypes.byref(c), _p(piv), _p(U), _p(L11), _p(L), n,
                              _p(ws), ws.numel(), _p(info), _stream(dev)))
    return piv, U, L11, L, Result(None, None, None, info).info()


def sketch_gauss(A: torch.Tensor, s: int, seed: int, stream_id: int, row0: int = 0) -> torch.Tensor:
    """Omega A with Omega's columns = global rows row0.. (R#19)."""
    _need(A, "A")
    rows, n = A.shape
    out = torch.empty(s, n, dtype=torch.float64, device=A.device)
    ws = _ws(lib().rlhc_sketch_gauss_workspace_size(rows, n, s), A.device)
    check(lib().rlhc_sketch_gauss(_p(A), rows, n, A.stride(0), row0, s, seed, stream_id, _p(out), _p(ws), ws.numel(),
                                  _stream(A.device)))
    return out


def sketch_count(A: torch.Tensor, s1: int, seed: int, row0: int = 0, want_hash: bool = False):
    """CountSketch Omega_1 A; optionally the (bucket, sign) of every row."""
    _need(A, "A")
    rows, n = A.shape
    out = torch.empty(s1, n, dtype=torch.float64, device=A.device)
    bucket = torch.empty(rows, dtype=torch.int32, device=A.device) if want_hash else None
    sign = torch.empty(rows, dtype=torch.int8, device=A.device) if want_hash else None
    ws = _ws(lib().rlhc_sketch_count_workspace_size(rows, n, s1), A.device)
    check(lib().rlhc_sketch_count(_p(A), rows, n, A.stride(0), row0, s1, seed, _p(out), _p(bucket), _p(sign), _p(ws),
                                  ws.numel(), _stream(A.device)))
    return (out, bucket, sign) if want_hash else out


def gram(A: torch.Tensor) -> torch.Tensor:
    """G = A^T A, exactly symmetric."""
    _need(A, "A")
    rows, n = A.shape
    G = torch.empty(n, n, dtype=torch.float64, device=A.device)
    ws = _ws(lib().rlhc_gram_workspace_size(rows, n), A.device)
    check(lib().rlhc_gram(_p(A), rows, n, A.stride(0), _p(G), _p(ws), ws.numel(), _stream(A.device)))
    return G


def trsm_apply(A: torch.Tensor, T: torch.Tensor, mode: int = RLHC_SUBST, out: torch.Tensor | None = None,
               want_gram: bool = False):
    """A T^{-1} for upper-triangular T; (out, G or None, info)."""
    _need(A, "A"); _need(T, "T")
    rows, n = A.shape
    out = torch.empty_like(A) if out is None else out
    G = torch.empty(n, n, dtype=torch.float64, device=A.device) if want_gram else None
    ws = _ws(lib().rlhc_trsm_apply_workspace_size(rows, n), A.device)
    info = _new_info(A.device)
    check(lib().rlhc_trsm_apply(_p(A), rows, n, A.stride(0), _p(T.contiguous()), mode, _p(out), out.stride(0), _p(G),
                                _p(ws), ws.numel(), _p(info), _stream(A.device)))
    return out, G, Result(None, None, None, info).info()


def hqr_r(A: torch.Tensor, sgn_ref: torch.Tensor | None = None):
    """Householder R of A (s x n), optional sign alignment with sgn_ref's diagonal."""
    _need(A, "A")
    s, n = A.shape
    S = torch.empty(n, n, dtype=torch.float64, device=A.device)
    ws = _ws(lib().rlhc_hqr_workspace_size(s, n), A.device)
    info = _new_info(A.device)
    check(lib().rlhc_hqr_r(_p(A), s, n, A.stride(0), _p(sgn_ref), _p(S), _p(ws), ws.numel(), _p(info),
                           _stream(A.device)))
    return S, Result(None, None, None, info).info()


def cholesky(G: torch.Tensor, stage: int = STAGE_CHOL1):
    """Upper Cholesky factor with breakdown reported as (code, stage, index)."""
    _need(G, "G")
    n = G.shape[0]
    Rm = torch.empty(n, n, dtype=torch.float64, device=G.device)
    info = _new_info(G.device)
    check(lib().rlhc_cholesky(_p(G.contiguous()), n, _p(Rm), stage, _p(info), _stream(G.device)))
    return Rm, Result(None, None, None, info).info()
