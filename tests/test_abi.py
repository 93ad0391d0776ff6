"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports every
symbol include/rlhc.h declares, and rejects invalid arguments on the host (no device
calls -- this container has no GPU)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "rlhc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rlhc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2412_06551_b200 import _lib
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    from paper_2412_06551_b200 import _lib
    names = _declared()
    assert "rlhc_slhc3" in names and "rlhc_sslhc3" in names and "rlhc_getrf_ts" in names
    for nm in names:
        assert hasattr(L, nm), nm
    assert sorted(_lib.EXPORTED) == names


def test_sm100a_cubin(L):
    import subprocess
    from paper_2412_06551_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core path present


def test_default_cfg_and_workspace(L):
    from paper_2412_06551_b200 import _lib
    c = _lib.TsluCfg()
    # the warp tournament's contract: 16-column panels, 128-row leaves, nodes of 8 children
    for (m, n, exp) in [(2048, 16, (128, 8, 16)), (65536, 64, (128, 8, 16)), (1 << 20, 128, (128, 8, 16)),
                        (262144, 512, (128, 8, 16)), (1000, 40, (128, 8, 16)), (100, 5, (128, 8, 5))]:
        L.rlhc_default_tslu_cfg(m, n, ctypes.byref(c))
        assert c.as_tuple() == exp, (m, n, c.as_tuple())
    assert L.rlhc_workspace_size(0, 65536, 64, 128, 0, None) > 0
    assert L.rlhc_workspace_size(1, 1 << 20, 128, 1024, 256, None) > 0
    assert L.rlhc_workspace_size(0, 65536, 64, 32, 0, None) == 0        # s < n
    assert L.rlhc_workspace_size(1, 65536, 64, 128, 256, None) == 0     # s2 > s1
    # exact GEPP: one leaf holding every row
    assert L.rlhc_workspace_size(0, 65536, 64, 128, 0, ctypes.byref(_lib.TsluCfg(65536, 2, 16))) > 0
    bad = _lib.TsluCfg(300, 4, 64)  # leaves larger than a select CTA holds
    assert L.rlhc_workspace_size(0, 65536, 64, 128, 0, ctypes.byref(bad)) == 0


def test_host_argument_errors(L):
    from paper_2412_06551_b200 import _lib
    info = ctypes.c_void_p(0x1000)
    fake = ctypes.c_void_p(0x10000)
    # null X
    rc = L.rlhc_slhc3(None, 100, 4, 4, 8, 0, None, fake, 4, fake, fake, fake, 1 << 20, info, None)
    assert rc == _lib.RLHC_EINVAL
    # m < n
    rc = L.rlhc_slhc3(fake, 3, 4, 4, 8, 0, None, ctypes.c_void_p(0x900000), 4, fake, fake, fake, 1 << 20, info, None)
    assert rc == _lib.RLHC_EINVAL
    # Q overlapping X
    rc = L.rlhc_slhc3(fake, 100, 4, 4, 8, 0, None, ctypes.c_void_p(0x10000 + 64), 4, fake, fake,
                      ctypes.c_void_p(0x100000), 1 << 24, info, None)
    assert rc == _lib.RLHC_EINVAL
    assert b"overlap" in L.rlhc_last_error()
    # workspace too small
    rc = L.rlhc_slhc3(fake, 100, 4, 4, 8, 0, None, ctypes.c_void_p(0x900000), 4, fake, fake,
                      ctypes.c_void_p(0x100000), 16, info, None)
    assert rc == _lib.RLHC_EWORKSPACE
    assert L.rlhc_version().startswith(b"rlhc-b200")


def test_dist_entry_host_errors():
    """rlhc_slhc3_dist argument checks are host-side (no GPU needed): bad shards, nulls."""
    import ctypes
    from paper_2412_06551_b200 import _lib
    L = _lib.lib()
    cfg = _lib.TsluCfg(256, 4, 64)
    dummy = ctypes.c_void_p(256)
    info = ctypes.c_void_p(512)
    # one rank (no communicator) must hold all rows
    rc = L.rlhc_slhc3_dist(dummy, 4096, 64, 64, 0, 8192, 128, ctypes.c_uint64(1), ctypes.byref(cfg), dummy, 64, dummy,
                           dummy, dummy, 1 << 30, info, None, None)
    assert rc == _lib.RLHC_EINVAL and b"shards" in L.rlhc_last_error()
    rc = L.rlhc_slhc3_dist(None, 4096, 64, 64, 0, 4096, 128, ctypes.c_uint64(1), ctypes.byref(cfg), dummy, 64, dummy,
                           dummy, dummy, 1 << 30, info, None, None)
    assert rc == _lib.RLHC_EINVAL
    # the contract is validated before any arithmetic on it (leaf_rows = 0 used to divide by
    # zero, arity 1 to loop forever)
    for bad in (_lib.TsluCfg(0, 4, 64), _lib.TsluCfg(256, 1, 64), _lib.TsluCfg(256, 4, 0)):
        rc = L.rlhc_sslhc3_dist(dummy, 4096, 64, 64, 0, 4096, 512, 128, ctypes.c_uint64(1), ctypes.byref(bad), dummy,
                                64, dummy, dummy, dummy, 1 << 30, info, None, None)
        assert rc == _lib.RLHC_EINVAL and b"configuration" in L.rlhc_last_error()
        assert L.rlhc_dist_workspace_size(0, 65536, 64, 128, 0, ctypes.byref(bad), 8) == 0
    assert L.rlhc_dist_workspace_size(0, 65536, 64, 128, 0, ctypes.byref(cfg), 8) > 0


def test_host_pipeline_host_checks(L):
    """rlhc_host_pipeline: workspace = the algorithm's plus two device copies of X, Q, R, piv,
    info; invalid algorithm / sizes / pointers are host errors (no device call)."""
    from paper_2412_06551_b200 import _lib
    m, n, s = 4096, 32, 64
    cfg = _lib.TsluCfg()
    L.rlhc_default_tslu_cfg(m, n, ctypes.byref(cfg))
    algo_ws = L.rlhc_workspace_size(0, m, n, s, 0, ctypes.byref(cfg))
    ws = L.rlhc_host_pipeline_workspace_size(0, m, n, s, 0, ctypes.byref(cfg))
    assert ws >= algo_ws + 2 * 8 * (2 * m * n + n * n + n)
    assert L.rlhc_host_pipeline_workspace_size(0, m, n, n - 1, 0, ctypes.byref(cfg)) == 0  # s < n
    assert L.rlhc_host_pipeline(7, 0, None, m, n, s, 0, None, ctypes.byref(cfg), None, None, None, None, None,
                                0, None) == _lib.RLHC_EINVAL
    assert L.rlhc_host_pipeline(0, 1, None, m, n, s, 0, None, ctypes.byref(cfg), None, None, None, None, None,
                                0, None) == _lib.RLHC_EINVAL
