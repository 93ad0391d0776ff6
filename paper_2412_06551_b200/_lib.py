"""ctypes binding of include/rlhc.h (argument marshalling only).

The library is built in-tree (paper_2412_06551_b200/librlhc.so).  There is no CPU
fallback: loading fails loudly when the library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librlhc.so")

# enum rlhc_code / rlhc_stage / rlhc_algo / rlhc_trsm_mode (include/rlhc.h)
(RLHC_OK, RLHC_EINVAL, RLHC_ENONFINITE, RLHC_ERANKDEF, RLHC_ESINGULAR, RLHC_EBREAKDOWN, RLHC_ECUDA, RLHC_EWORKSPACE,
 RLHC_ENCCL) = range(9)
(STAGE_INPUT, STAGE_LU, STAGE_SKETCH, STAGE_HQR, STAGE_SOLVE_Y, STAGE_CHOL1, STAGE_SOLVE_D, STAGE_CHOL2,
 STAGE_SOLVE_J, STAGE_CHOL0) = range(10)
RLHC_SLHC3, RLHC_SSLHC3 = 0, 1
RLHC_CHOLQR2, RLHC_SCHOLQR3, RLHC_LUC2, RLHC_RHC = 2, 3, 4, 5
RLHC_SUBST, RLHC_INV_GEMM = 0, 1

CODE_NAMES = {0: "OK", 1: "EINVAL", 2: "ENONFINITE", 3: "ERANKDEF", 4: "ESINGULAR", 5: "EBREAKDOWN", 6: "ECUDA",
              7: "EWORKSPACE", 8: "ENCCL"}
STAGE_NAMES = {0: "INPUT", 1: "LU", 2: "SKETCH", 3: "HQR", 4: "SOLVE_Y", 5: "CHOL1", 6: "SOLVE_D", 7: "CHOL2",
               8: "SOLVE_J", 9: "CHOL0"}


class TsluCfg(ctypes.Structure):
    _fields_ = [("leaf_rows", ctypes.c_int64), ("arity", ctypes.c_int32), ("panel", ctypes.c_int32)]

    def as_tuple(self):
        return int(self.leaf_rows), int(self.arity), int(self.panel)


class Info(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("stage", ctypes.c_int32), ("index", ctypes.c_int64)]


_lib = None


def lib():
    """Load librlhc.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    try:
        _build.build()
    except Exception as e:  # pragma: no cover - no nvcc on the target is fatal only when stale
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librlhc.so is missing and could not be built: {e}") from e
    L = ctypes.CDLL(LIB_PATH)
    P, I64, U64, U32, SZ, I = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t,
                               ctypes.c_int)
    PC = ctypes.POINTER(TsluCfg)
    L.rlhc_tslw_schur.argtypes = [P, I64, I64, I64, P, I64, I64, P, P]
    L.rlhc_tslw_schur_reduce_to.argtypes = [P, I64, I64, I64, P, I64, I64, I64, P, P, PC, I64, P, P, P, P, SZ, P]
    L.rlhc_tslw_owned_rows.argtypes = [P, I64, P, I64, I64, I64, P, I64, I64, I64, P, P, P]
    L.rlhc_tslw_finish.argtypes = [P, I64, I64, I64, I64, P, P, P]
    L.rlhc_host_pipeline_workspace_size.argtypes = [I, I64, I64, I64, I64, PC]
    L.rlhc_host_pipeline_workspace_size.restype = SZ
    L.rlhc_host_pipeline.argtypes = [I, I64, P, I64, I64, I64, I64, P, PC, P, P, P, P, P, SZ, P]
    L.rlhc_graph_begin.argtypes = [P]
    L.rlhc_graph_end.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
    L.rlhc_graph_launch.argtypes = [P, P]
    L.rlhc_graph_destroy.argtypes = [P]
    L.rlhc_graph_destroy.restype = None
    L.rlhc_default_tslu_cfg.argtypes = [I64, I64, PC]
    L.rlhc_default_tslu_cfg.restype = None
    L.rlhc_workspace_size.argtypes = [I, I64, I64, I64, I64, PC]
    L.rlhc_workspace_size.restype = SZ
    L.rlhc_slhc3.argtypes = [P, I64, I64, I64, I64, U64, PC, P, I64, P, P, P, SZ, P, P]
    L.rlhc_sslhc3.argtypes = [P, I64, I64, I64, I64, I64, U64, PC, P, I64, P, P, P, SZ, P, P]
    L.rlhc_getrf_ts_workspace_size.argtypes = [I64, I64, PC]
    L.rlhc_getrf_ts_workspace_size.restype = SZ
    L.rlhc_getrf_ts.argtypes = [P, I64, I64, I64, I64, PC, P, P, P, P, I64, P, SZ, P, P]
    L.rlhc_sketch_gauss_workspace_size.argtypes = [I64, I64, I64]
    L.rlhc_sketch_gauss_workspace_size.restype = SZ
    L.rlhc_sketch_gauss.argtypes = [P, I64, I64, I64, I64, I64, U64, U32, P, P, SZ, P]
    L.rlhc_sketch_count_workspace_size.argtypes = [I64, I64, I64]
    L.rlhc_sketch_count_workspace_size.restype = SZ
    L.rlhc_sketch_count.argtypes = [P, I64, I64, I64, I64, I64, U64, P, P, P, P, SZ, P]
    L.rlhc_gram_workspace_size.argtypes = [I64, I64]
    L.rlhc_gram_workspace_size.restype = SZ
    L.rlhc_gram.argtypes = [P, I64, I64, I64, P, P, SZ, P]
    L.rlhc_trsm_apply_workspace_size.argtypes = [I64, I64]
    L.rlhc_trsm_apply_workspace_size.restype = SZ
    L.rlhc_trsm_apply.argtypes = [P, I64, I64, I64, P, I, P, I64, P, P, SZ, P, P]
    L.rlhc_hqr_workspace_size.argtypes = [I64, I64]
    L.rlhc_hqr_workspace_size.restype = SZ
    L.rlhc_hqr_r.argtypes = [P, I64, I64, I64, P, P, P, SZ, P, P]
    L.rlhc_cholesky.argtypes = [P, I64, P, I, P, P]
    L.rlhc_version.restype = ctypes.c_char_p
    L.rlhc_last_error.restype = ctypes.c_char_p
    # row-sharded building blocks
    L.rlhc_tslu_local_workspace_size.argtypes = [I64, I64, PC]
    L.rlhc_tslu_local_workspace_size.restype = SZ
    L.rlhc_tslu_reduce.argtypes = [P, I64, I64, I64, I64, I64, P, PC, P, P, P, P, SZ, P]
    L.rlhc_tslu_reduce_to.argtypes = [P, I64, I64, I64, I64, I64, P, PC, I64, P, P, P, P, SZ, P]
    L.rlhc_tslu_reduce_to.restype = I
    L.rlhc_tslu_local_slots.argtypes = [I64, PC]
    L.rlhc_tslu_local_slots.restype = I64
    L.rlhc_tslu_combine.argtypes = [P, P, P, I64, I64, PC, P, P, P, P, SZ, P]
    L.rlhc_owned_rows.argtypes = [P, I64, I64, I64, P, P, I64, I64, I64, P, P]
    L.rlhc_tslu_panel_workspace_size.argtypes = [I64]
    L.rlhc_tslu_panel_workspace_size.restype = SZ
    L.rlhc_tslu_panel_factor_rows.argtypes = [P, P, I64, I64, I64, I64, I64, P, P, P, P, SZ, P, P]
    L.rlhc_tslu_eliminate_workspace_size.argtypes = [I64]
    L.rlhc_tslu_eliminate_workspace_size.restype = SZ
    L.rlhc_tslu_eliminate.argtypes = [P, I64, I64, I64, I64, I64, P, P, I64, P, SZ, P]
    L.rlhc_lfactor_workspace_size.argtypes = [I64, I64]
    L.rlhc_lfactor_workspace_size.restype = SZ
    L.rlhc_l11.argtypes = [P, I64, P, P, P, SZ, P]
    L.rlhc_lfactor.argtypes = [P, I64, I64, I64, I64, P, P, P, P, I64, P, SZ, P]
    L.rlhc_trmm_upper.argtypes = [P, P, I64, P, P]
    L.rlhc_cholesky_workspace_size.argtypes = [I64]
    L.rlhc_cholesky_workspace_size.restype = SZ
    L.rlhc_cholesky_ws.argtypes = [P, I64, P, I, P, SZ, P, P]
    for name in ("rlhc_tslu_reduce", "rlhc_tslu_combine", "rlhc_owned_rows", "rlhc_tslu_panel_factor_rows",
                 "rlhc_tslu_eliminate", "rlhc_l11", "rlhc_lfactor", "rlhc_trmm_upper", "rlhc_cholesky_ws"):
        getattr(L, name).restype = I
    L.rlhc_launch_count.restype = ctypes.c_uint64
    L.rlhc_stage_timing.argtypes = [I]
    L.rlhc_stage_timing.restype = None
    L.rlhc_stage_times.argtypes = [P, I]
    L.rlhc_stage_times.restype = I
    L.rlhc_stage_name.argtypes = [I]
    L.rlhc_stage_name.restype = ctypes.c_char_p
    for name in ("rlhc_slhc3", "rlhc_sslhc3", "rlhc_getrf_ts", "rlhc_sketch_gauss", "rlhc_sketch_count", "rlhc_gram",
                 "rlhc_trsm_apply", "rlhc_hqr_r", "rlhc_cholesky"):
        getattr(L, name).restype = I
    # the paper's comparison algorithms
    L.rlhc_method_workspace_size.argtypes = [I, I64, I64, I64, I64, PC]
    L.rlhc_method_workspace_size.restype = SZ
    L.rlhc_cholqr2.argtypes = [P, I64, I64, I64, P, I64, P, P, SZ, P, P]
    L.rlhc_scholqr3.argtypes = [P, I64, I64, I64, P, I64, P, P, SZ, P, P]
    L.rlhc_luc2.argtypes = [P, I64, I64, I64, PC, P, I64, P, P, P, SZ, P, P]
    L.rlhc_rhc.argtypes = [P, I64, I64, I64, I64, I64, ctypes.c_uint64, P, I64, P, P, SZ, P, P]
    for name in ("rlhc_cholqr2", "rlhc_scholqr3", "rlhc_luc2", "rlhc_rhc"):
        getattr(L, name).restype = I
    # row-sharded entry points over NCCL
    L.rlhc_comm_unique_id.argtypes = [P]
    L.rlhc_comm_init.argtypes = [ctypes.POINTER(P), I, I, P]
    L.rlhc_comm_destroy.argtypes = [P]
    for name in ("rlhc_comm_unique_id", "rlhc_comm_init", "rlhc_comm_destroy", "rlhc_slhc3_dist", "rlhc_sslhc3_dist"):
        getattr(L, name).restype = I
    L.rlhc_dist_workspace_size.argtypes = [I, I64, I64, I64, I64, PC, I]
    L.rlhc_dist_workspace_size.restype = SZ
    L.rlhc_slhc3_dist.argtypes = [P, I64, I64, I64, I64, I64, I64, ctypes.c_uint64, PC, P, I64, P, P, P, SZ, P, P, P]
    L.rlhc_sslhc3_dist.argtypes = [P, I64, I64, I64, I64, I64, I64, I64, ctypes.c_uint64, PC, P, I64, P, P, P, SZ, P, P,
                                   P]
    _lib = L
    return L


# Every symbol include/rlhc.h declares (checked by tests/test_abi.py).
EXPORTED = ["rlhc_default_tslu_cfg", "rlhc_workspace_size", "rlhc_slhc3", "rlhc_sslhc3",
            "rlhc_getrf_ts_workspace_size", "rlhc_getrf_ts", "rlhc_sketch_gauss_workspace_size",
            "rlhc_sketch_gauss", "rlhc_sketch_count_workspace_size", "rlhc_sketch_count",
            "rlhc_gram_workspace_size", "rlhc_gram", "rlhc_trsm_apply_workspace_size", "rlhc_trsm_apply",
            "rlhc_hqr_workspace_size", "rlhc_hqr_r", "rlhc_cholesky", "rlhc_version", "rlhc_last_error",
            "rlhc_launch_count", "rlhc_stage_timing", "rlhc_stage_times", "rlhc_stage_name",
            "rlhc_tslu_local_workspace_size", "rlhc_tslu_reduce", "rlhc_tslu_reduce_to", "rlhc_tslu_local_slots",
            "rlhc_tslu_combine", "rlhc_owned_rows",
            "rlhc_tslu_panel_workspace_size", "rlhc_tslu_panel_factor_rows", "rlhc_tslu_eliminate_workspace_size",
            "rlhc_tslu_eliminate", "rlhc_lfactor_workspace_size", "rlhc_l11", "rlhc_lfactor", "rlhc_trmm_upper",
            "rlhc_cholesky_workspace_size", "rlhc_cholesky_ws", "rlhc_comm_unique_id", "rlhc_comm_init",
            "rlhc_comm_destroy", "rlhc_dist_workspace_size", "rlhc_slhc3_dist", "rlhc_sslhc3_dist",
            "rlhc_method_workspace_size", "rlhc_cholqr2", "rlhc_scholqr3", "rlhc_luc2", "rlhc_rhc",
            "rlhc_graph_begin", "rlhc_graph_end", "rlhc_graph_launch", "rlhc_graph_destroy",
            "rlhc_tslw_schur", "rlhc_tslw_schur_reduce_to", "rlhc_tslw_owned_rows", "rlhc_tslw_finish",
            "rlhc_host_pipeline_workspace_size", "rlhc_host_pipeline"]
NUM_TIMED_STAGES = 13


def stage_times(reset: bool = True) -> dict:
    """Per-stage milliseconds accumulated by rlhc_stage_timing (synchronises)."""
    buf = (ctypes.c_double * NUM_TIMED_STAGES)()
    calls = lib().rlhc_stage_times(buf, NUM_TIMED_STAGES)
    if calls < 0:
        raise RlhcError(RLHC_ECUDA, "stage timing events failed")
    names = [lib().rlhc_stage_name(k).decode() for k in range(NUM_TIMED_STAGES)]
    return {"calls": calls, **{nm: buf[k] for k, nm in enumerate(names)}}


class RlhcError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"rlhc {CODE_NAMES.get(code, code)}: {msg}")
        self.code = code


def check(rc: int):
    if rc != RLHC_OK:
        raise RlhcError(rc, lib().rlhc_last_error().decode())
