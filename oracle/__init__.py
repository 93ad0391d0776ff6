"""CPU fp64 oracle for SLHC3 / SSLHC3 (arXiv 2412.06551) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It shares no code with the CUDA
path (``paper_2412_06551_b200``) and never imports it.  The arithmetic lives in
``rlhc_oracle.c`` (plain C, ``-ffp-contract=off``); this module only marshals numpy
arrays through ctypes.  Every C function cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rlhc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# error codes / stages, declared independently of include/rlhc.h (SURVEY 8b numbering)
OK, EINVAL, ENONFINITE, ERANKDEF, ESINGULAR, EBREAKDOWN = 0, 1, 2, 3, 4, 5
ST_INPUT, ST_LU, ST_SKETCH, ST_HQR, ST_SOLVE_Y, ST_CHOL1, ST_SOLVE_D, ST_CHOL2, ST_SOLVE_J, ST_CHOL0 = range(10)


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, fp64, no fp contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        # -mfma only lets fma() compile to the instruction (it is exact either way); with
        # -ffp-contract=off no a*b+c is ever contracted, so the arithmetic is unchanged
        isa = ["-mfma", "-mavx2"] if _host_has_fma() else []
        subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", *isa, "-fopenmp", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _host_has_fma() -> bool:
    try:
        return any(" fma " in f" {ln.split(":", 1)[1]} " and " avx2 " in f" {ln.split(":", 1)[1]} "
                   for ln in open("/proc/cpuinfo") if ln.startswith("flags"))
    except OSError:
        return False


class _Info(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("stage", ctypes.c_int32), ("index", ctypes.c_int64)]


class _Stages(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("U", "L11", "Lt", "Ls", "S", "Y", "G1", "D", "G2", "J")]


_lib = None
_ROWS_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double))
_QROWS_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double))


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P, I64, U64, U32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double
        L.ora_philox.argtypes = [P, P, P]
        L.ora_det_log.argtypes = [D]; L.ora_det_log.restype = D
        L.ora_det_sincos2pi.argtypes = [D, P, P]
        L.ora_gauss_pair.argtypes = [U64, U64, U32, U32, P, P]
        L.ora_omega.argtypes = [U64, U32, I64, I64, I64]; L.ora_omega.restype = D
        L.ora_omega_block.argtypes = [U64, U32, I64, I64, I64, P]
        L.ora_cs_hash.argtypes = [U64, I64, I64, I64, P, P]
        L.ora_cs_apply.argtypes = [P, I64, I64, I64, P, P, I64, P]
        L.ora_sketch_gauss.argtypes = [P, I64, I64, I64, I64, I64, U64, U32, P]
        L.ora_tslu.argtypes = [P, I64, I64, I64, I64, I64, I64, P, P, P, P, P]
        L.ora_lfactor.argtypes = [P, I64, I64, I64, P, P, P, P]
        L.ora_hqr_r.argtypes = [P, I64, I64, P, P]
        L.ora_trmm_uu.argtypes = [P, P, I64, P]
        L.ora_trsm_right_upper.argtypes = [P, I64, I64, I64, P, P, I64, ctypes.c_int, P]
        L.ora_gram.argtypes = [P, I64, I64, I64, P]
        L.ora_chol.argtypes = [P, I64, P, ctypes.c_int, P]
        L.ora_slhc3.argtypes = [P, I64, I64, I64, I64, U64, I64, I64, I64, P, I64, P, P, P, P]
        L.ora_sslhc3.argtypes = [P, I64, I64, I64, I64, I64, U64, I64, I64, I64, P, I64, P, P, P, P]
        L.ora_orthogonality.argtypes = [P, I64, I64, I64]; L.ora_orthogonality.restype = D
        L.ora_residual.argtypes = [P, P, P, I64, I64, I64, I64]; L.ora_residual.restype = D
        L.ora_num_threads.restype = ctypes.c_int
        L.ora_select.argtypes = [P, P, I64, I64, P]; L.ora_select.restype = I64
        L.ora_panel_rows.argtypes = [P, I64, I64]
        L.ora_eliminate_rows.argtypes = [P, I64, I64, I64, I64, P, P]
        L.ora_lfactor_rows.argtypes = [P, I64, I64, I64, P, P, P, P]
        L.ora_cholqr2.argtypes = [P, I64, I64, I64, P, I64, P, P]
        L.ora_scholqr3.argtypes = [P, I64, I64, I64, P, I64, P, P]
        L.ora_scholqr_shift.argtypes = [P, I64, I64]; L.ora_scholqr_shift.restype = D
        L.ora_luc2.argtypes = [P, I64, I64, I64, I64, I64, I64, P, I64, P, P, P]
        L.ora_rhc.argtypes = [P, I64, I64, I64, I64, I64, U64, P, I64, P, P]
        L.ora_lhc3_chunked.argtypes = [ctypes.c_int, I64, I64, I64, I64, U64, I64, I64, I64, I64, _ROWS_FN, _QROWS_FN,
                                       P, P, P, P, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, stage, index):
        super().__init__(f"oracle error code={code} stage={stage} index={index}")
        self.code, self.stage, self.index = code, stage, index


def _raise(info: _Info):
    if info.code:
        raise OracleError(info.code, info.stage, info.index)


# ----------------------------------------------------------------- RNG pieces
def philox(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32).copy(); k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().ora_philox(_p(c), _p(k), _p(out))
    return out


def det_log(x: float) -> float:
    return lib().ora_det_log(float(x))


def det_sincos2pi(u: float):
    s, c = ctypes.c_double(), ctypes.c_double()
    lib().ora_det_sincos2pi(float(u), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def gauss_pair(seed: int, j: int, c2: int, stream: int):
    z0, z1 = ctypes.c_double(), ctypes.c_double()
    lib().ora_gauss_pair(seed, j, c2, stream, ctypes.byref(z0), ctypes.byref(z1))
    return z0.value, z1.value


def omega_block(seed: int, stream: int, s: int, j0: int, cols: int) -> np.ndarray:
    out = np.zeros((s, cols))
    lib().ora_omega_block(seed, stream, s, j0, cols, _p(out))
    return out


def cs_hash(seed: int, row0: int, rows: int, s1: int):
    b = np.zeros(rows, np.int32); sg = np.zeros(rows, np.int8)
    lib().ora_cs_hash(seed, row0, rows, s1, _p(b), _p(sg))
    return b, sg


def cs_apply(A, bucket, sign, s1: int) -> np.ndarray:
    A = _f64(A); rows, n = A.shape
    b = np.ascontiguousarray(bucket, np.int32); sg = np.ascontiguousarray(sign, np.int8)
    out = np.zeros((s1, n))
    lib().ora_cs_apply(_p(A), rows, n, n, _p(b), _p(sg), s1, _p(out))
    return out


def sketch_gauss(A, s: int, seed: int, stream: int, row0: int = 0) -> np.ndarray:
    A = _f64(A); rows, n = A.shape
    out = np.zeros((s, n))
    lib().ora_sketch_gauss(_p(A), rows, n, n, row0, s, seed, stream, _p(out))
    return out


# ------------------------------------------------------------------- LU
def tslu(X, leaf_rows: int, arity: int, panel: int | None = None, want_L: bool = False):
    X = _f64(X); m, n = X.shape
    panel = n if panel is None else panel
    piv = np.zeros(n, np.int64); U = np.zeros((n, n)); L11 = np.zeros((n, n))
    L = np.zeros((m, n)) if want_L else None
    info = _Info()
    lib().ora_tslu(_p(X), m, n, n, leaf_rows, arity, panel, _p(piv), _p(U), _p(L11),
                   _p(L) if want_L else None, ctypes.byref(info))
    _raise(info)
    return (piv, U, L11, L) if want_L else (piv, U, L11)


def lfactor(X, piv, U, L11) -> np.ndarray:
    X = _f64(X); m, n = X.shape
    piv = np.ascontiguousarray(piv, np.int64); U = _f64(U); L11 = _f64(L11)
    L = np.zeros((m, n))
    lib().ora_lfactor(_p(X), m, n, n, _p(piv), _p(U), _p(L11), _p(L))
    return L


# ------------------------------------------------------------- dense kernels
def hqr_r(A) -> np.ndarray:
    A = _f64(A).copy(); s, n = A.shape
    R = np.zeros((n, n)); info = _Info()
    lib().ora_hqr_r(_p(A), s, n, _p(R), ctypes.byref(info))
    _raise(info)
    return R


def trmm_uu(A, B) -> np.ndarray:
    A = _f64(A); B = _f64(B); n = A.shape[0]
    C = np.zeros((n, n))
    lib().ora_trmm_uu(_p(A), _p(B), n, _p(C))
    return C


def trsm_right_upper(A, T, stage: int = ST_SOLVE_Y) -> np.ndarray:
    A = _f64(A); T = _f64(T); rows, n = A.shape
    out = np.zeros((rows, n)); info = _Info()
    lib().ora_trsm_right_upper(_p(A), rows, n, n, _p(T), _p(out), n, stage, ctypes.byref(info))
    _raise(info)
    return out


def gram(A) -> np.ndarray:
    A = _f64(A); rows, n = A.shape
    G = np.zeros((n, n))
    lib().ora_gram(_p(A), rows, n, n, _p(G))
    return G


def chol(G, stage: int = ST_CHOL1) -> np.ndarray:
    G = _f64(G); n = G.shape[0]
    R = np.zeros((n, n)); info = _Info()
    lib().ora_chol(_p(G), n, _p(R), stage, ctypes.byref(info))
    _raise(info)
    return R


# -------------------------------------------------------------- algorithms
@dataclass
class Result:
    Q: np.ndarray
    R: np.ndarray
    piv: np.ndarray
    stages: dict
    info: tuple  # (code, stage, index)


_STAGE_SHAPES = ("U", "L11", "Lt", "Ls", "S", "Y", "G1", "D", "G2", "J")


def _run(fn, X, n, args, s_rows, s1_rows, stages: bool, raise_on_error: bool):
    X = _f64(X); m = X.shape[0]
    Q = np.zeros((m, n)); R = np.zeros((n, n)); piv = np.zeros(n, np.int64)
    info = _Info()
    st = _Stages(); arrs = {}
    if stages:
        for k in _STAGE_SHAPES:
            shape = (s_rows, n) if k == "Ls" else (s1_rows, n) if k == "Lt" else (n, n)
            if k == "Lt" and s1_rows is None:
                continue
            arrs[k] = np.zeros(shape)
            setattr(st, k, arrs[k].ctypes.data)
    fn(_p(X), m, n, n, *args, _p(Q), n, _p(R), _p(piv), ctypes.byref(st), ctypes.byref(info))
    if raise_on_error:
        _raise(info)
    return Result(Q, R, piv, arrs, (info.code, info.stage, info.index))


def slhc3(X, s: int, seed: int, leaf_rows: int, arity: int, panel: int | None = None, stages: bool = False,
          raise_on_error: bool = True) -> Result:
    n = X.shape[1]
    panel = n if panel is None else panel
    return _run(lib().ora_slhc3, X, n, (s, seed, leaf_rows, arity, panel), s, None, stages, raise_on_error)


def sslhc3(X, s1: int, s2: int, seed: int, leaf_rows: int, arity: int, panel: int | None = None,
           stages: bool = False, raise_on_error: bool = True) -> Result:
    n = X.shape[1]
    panel = n if panel is None else panel
    return _run(lib().ora_sslhc3, X, n, (s1, s2, seed, leaf_rows, arity, panel), s2, s1, stages, raise_on_error)


def lhc3_chunked(algo: str, m: int, n: int, get_rows, s_or_s1: int, s2: int, seed: int, leaf_rows: int, arity: int,
                 panel: int, chunk_rows: int = 65536, put_q=None, stages: bool = False,
                 raise_on_error: bool = True) -> Result:
    """SLHC3 / SSLHC3 with X streamed in row chunks (ora_lhc3_chunked; cfg5 does not fit the
    in-memory oracle): get_rows(row0, rows) -> (rows x n) float64 array of X's rows;
    put_q(row0, Q_rows) (optional) receives Q's rows.  Bit-identical to slhc3 / sslhc3.
    Result.Q is None."""
    sslhc = algo == "sslhc3"
    R = np.zeros((n, n)); piv = np.zeros(n, np.int64); info = _Info()
    err = []

    def _get(user, row0, rows, buf):
        try:
            a = np.ascontiguousarray(get_rows(int(row0), int(rows)), dtype=np.float64)
            assert a.shape == (rows, n), a.shape
            ctypes.memmove(buf, a.ctypes.data, a.nbytes)
        except BaseException as e:  # noqa: BLE001 -- reported after the call
            err.append(e)

    def _put(user, row0, rows, buf):
        try:
            put_q(int(row0), np.ctypeslib.as_array(buf, shape=(int(rows), n)).copy())
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    cb_get = _ROWS_FN(_get)
    cb_put = _QROWS_FN(_put) if put_q is not None else _QROWS_FN()
    st = _Stages(); arrs = {}
    if stages:
        srows = s2 if sslhc else s_or_s1
        for k in _STAGE_SHAPES:
            if k == "Lt" and not sslhc:
                continue
            shape = (srows, n) if k == "Ls" else (s_or_s1, n) if k == "Lt" else (n, n)
            arrs[k] = np.zeros(shape)
            setattr(st, k, arrs[k].ctypes.data)
    lib().ora_lhc3_chunked(1 if sslhc else 0, m, n, s_or_s1, s2, ctypes.c_uint64(seed), leaf_rows, arity, panel,
                           chunk_rows, cb_get, cb_put, None, _p(R), _p(piv), ctypes.byref(st), ctypes.byref(info))
    if err:
        raise err[0]
    if raise_on_error:
        _raise(info)
    return Result(None, R, piv, arrs, (info.code, info.stage, info.index))


# -------------------------------------------------- comparison algorithms
def _run_simple(call, X, n, raise_on_error: bool):
    X = _f64(X); m = X.shape[0]
    Q = np.zeros((m, n)); R = np.zeros((n, n)); piv = np.zeros(n, np.int64)
    info = _Info()
    call(X, m, Q, R, piv, info)
    if raise_on_error:
        _raise(info)
    return Result(Q, R, piv, {}, (info.code, info.stage, info.index))


def cholqr2(X, raise_on_error: bool = True) -> Result:
    """CholeskyQR2 (alg:cholqr2)."""
    n = X.shape[1]
    return _run_simple(lambda X, m, Q, R, piv, info: lib().ora_cholqr2(_p(X), m, n, n, _p(Q), n, _p(R),
                                                                      ctypes.byref(info)), X, n, raise_on_error)


def scholqr3(X, raise_on_error: bool = True) -> Result:
    """SCholeskyQR3 (alg:Shifted3), shift of P:984 (R#21)."""
    n = X.shape[1]
    return _run_simple(lambda X, m, Q, R, piv, info: lib().ora_scholqr3(_p(X), m, n, n, _p(Q), n, _p(R),
                                                                       ctypes.byref(info)), X, n, raise_on_error)


def scholqr_shift(G, m: int) -> float:
    G = _f64(G)
    return lib().ora_scholqr_shift(_p(G), m, G.shape[0])


def luc2(X, leaf_rows: int, arity: int, panel: int | None = None, raise_on_error: bool = True) -> Result:
    """LU-CholeskyQR2 (alg:LU2) under the tournament contract."""
    n = X.shape[1]
    panel = n if panel is None else panel
    return _run_simple(lambda X, m, Q, R, piv, info: lib().ora_luc2(_p(X), m, n, n, leaf_rows, arity, panel, _p(Q), n,
                                                                   _p(R), _p(piv), ctypes.byref(info)),
                       X, n, raise_on_error)


def rhc(X, s1: int, s2: int, seed: int, raise_on_error: bool = True) -> Result:
    """Rand.Householder-Cholesky (alg:Rand2), multi-sketch K = Omega_2 Omega_1 X."""
    n = X.shape[1]
    return _run_simple(lambda X, m, Q, R, piv, info: lib().ora_rhc(_p(X), m, n, n, s1, s2, ctypes.c_uint64(seed),
                                                                  _p(Q), n, _p(R), ctypes.byref(info)),
                       X, n, raise_on_error)


def orthogonality(Q) -> float:
    Q = _f64(Q); m, n = Q.shape
    return lib().ora_orthogonality(_p(Q), m, n, n)


def residual(Q, R, X) -> float:
    Q = _f64(Q); R = _f64(R); X = _f64(X); m, n = Q.shape
    return lib().ora_residual(_p(Q), _p(R), _p(X), m, n, n, n)


# ---- pieces for the row-sharded orchestration check (tests/test_dist_cpu.py)
def select(B, ids, w: int):
    """GEPP selection on candidate rows B (cnt x w) with global ids: winners in pivot order."""
    B = _f64(B).copy(); ids = np.ascontiguousarray(ids, np.int64)
    out = np.zeros(max(w, 1), np.int64)
    k = lib().ora_select(_p(B), _p(ids), len(ids), w, _p(out))
    return out[:k]


def panel_rows(prow):
    prow = _f64(prow).copy(); w, ncols = prow.shape
    lib().ora_panel_rows(_p(prow), w, ncols)
    return prow


def eliminate_rows(A, p0: int, w: int, U, chosen):
    A = _f64(A); U = _f64(U); rows, n = A.shape
    ch = np.ascontiguousarray(chosen, np.uint8)
    lib().ora_eliminate_rows(_p(A), rows, n, p0, w, _p(U), _p(ch))
    return A


def lfactor_rows(X, row0: int, piv, U, L11):
    X = _f64(X); rows, n = X.shape
    piv = np.ascontiguousarray(piv, np.int64); U = _f64(U); L11 = _f64(L11)
    L = np.zeros((rows, n))
    lib().ora_lfactor_rows(_p(X), rows, n, row0, _p(piv), _p(U), _p(L11), _p(L))
    return L


def num_threads() -> int:
    return lib().ora_num_threads()
