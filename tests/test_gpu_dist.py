"""GPU checks of the row-sharded path (paper_2412_06551_b200.dist) through the C ABI:
world size 1 against the single-call pipeline, and world size 2 over gloo (both ranks on
cuda:0; gloo collectives are host-mediated, so no kernel waits on another rank) against
the oracle."""
import os
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def test_world1_matches_single_call(ora):
    import paper_2412_06551_b200 as rl
    import synth
    from paper_2412_06551_b200._lib import TsluCfg
    from paper_2412_06551_b200.dist import DistPlan
    for algo, m, n, kw, cfgt in [("sslhc3", 65536, 64, dict(s1=512, s2=128), (256, 2, 64)),
                                 ("slhc3", 32768, 32, dict(s=64), (512, 2, 32)),
                                 ("sslhc3", 16384, 100, dict(s1=800, s2=200), (256, 2, 64)),
                                 # the default (warp) contract: left-looking row-sharded panels
                                 ("slhc3", 65536, 64, dict(s=128), (128, 8, 16)),
                                 ("sslhc3", 16384, 100, dict(s1=800, s2=200), (128, 8, 16))]:
        X = synth.baseline_matrix(m, n, 10, 7, device="cuda")
        cfg = TsluCfg(*cfgt)
        plan = DistPlan(algo, m, n, seed=2, cfg=cfg, device="cuda", **kw)
        Q, R, piv, infos = plan.run(X)
        assert plan.first_error(infos) == (0, 0, 0)
        single = (rl.slhc3 if algo == "slhc3" else rl.sslhc3)(X, seed=2, cfg=cfg, **kw)
        assert torch.equal(piv, single.piv)
        Rh, Rs = R.cpu().numpy(), single.R.cpu().numpy()
        assert np.linalg.norm(Rh - Rs) <= 1e-12 * np.linalg.norm(Rs)
        Qh = Q.cpu().numpy()
        assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) <= 1e-13 * np.sqrt(n)


def _worker(rank, world, port, out_path, cfgt, m):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2412_06551_b200._lib import TsluCfg
        from paper_2412_06551_b200.dist import DistPlan
        n = 48
        cfg = TsluCfg(*cfgt)
        mloc = m // world
        X = synth.baseline_matrix(m, n, 9, 4, device="cuda", row0=rank * mloc, rows=mloc)
        plan = DistPlan("sslhc3", m, n, s1=384, s2=96, seed=6, cfg=cfg, device="cuda")
        Q, R, piv, infos = plan.run(X)
        torch.cuda.synchronize()
        np.savez(out_path + f".{rank}.npz", Q=Q.cpu().numpy(), R=R.cpu().numpy(), piv=piv.cpu().numpy(),
                 info=np.array(plan.first_error(infos)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfgt,m", [((256, 2, 48), 32768),
                                    ((128, 8, 16), 131072),    # 512 = 8^3 leaves per rank: one subtree
                                    ((128, 8, 16), 262144),    # 1024 leaves per rank: two subtrees (K = 2)
                                    ((128, 8, 16), 98304)])    # 384 leaves per rank: 6 level-2 subtrees
def test_two_gloo_ranks_on_one_gpu(ora, cfgt, m):
    """Two gloo ranks driving the CUDA stage calls on one GPU (the N > 1 orchestration of
    dist.py); each rank's rows are K >= 1 complete subtrees of the global tree, so the pivots
    are the single-process contract's."""
    import synth
    d = tempfile.mkdtemp()
    out = os.path.join(d, "r")
    mp.spawn(_worker, args=(2, 29700 + os.getpid() % 200 + (m >> 12) % 97, out, cfgt, m), nprocs=2, join=True)
    res = [np.load(out + f".{r}.npz") for r in range(2)]
    X = synth.baseline_matrix(m, 48, 9, 4, device="cuda").cpu().numpy()
    ref = ora.sslhc3(X, 384, 96, 6, *cfgt)
    for r in res:
        assert tuple(r["info"]) == (0, 0, 0)
        assert np.array_equal(r["piv"], ref.piv)
        assert np.linalg.norm(r["R"] - ref.R) <= 1e-12 * np.linalg.norm(ref.R)
    Q = np.concatenate([r["Q"] for r in res])
    assert np.linalg.norm(Q.T @ Q - np.eye(48)) <= 1e-13 * np.sqrt(48)


@pytest.mark.parametrize("with_comm", [False, True])
def test_c_dist_entry_matches_single_call(with_comm):
    """rlhc_slhc3_dist / rlhc_sslhc3_dist (C orchestration, NCCL collectives) on one rank: no
    communicator, and a real one-rank NCCL communicator; against the single-GPU call."""
    import paper_2412_06551_b200 as rl
    import synth
    from paper_2412_06551_b200._lib import TsluCfg
    from paper_2412_06551_b200.dist import CDistPlan, NcclComm
    comm = NcclComm() if with_comm else None
    for algo, m, n, kw, cfgt in [("slhc3", 65536, 64, dict(s=128), (256, 4, 64)),
                                 ("sslhc3", 65536, 128, dict(s1=1024, s2=256), (256, 4, 64)),
                                 ("sslhc3", 16384, 100, dict(s1=800, s2=200), (256, 2, 64)),
                                 ("slhc3", 65536, 64, dict(s=128), (128, 8, 16)),
                                 ("sslhc3", 65536, 128, dict(s1=1024, s2=256), (128, 8, 16))]:
        X = synth.baseline_matrix(m, n, 12, 8, device="cuda")
        cfg = TsluCfg(*cfgt)
        plan = CDistPlan(algo, m, n, seed=3, cfg=cfg, device="cuda", comm=comm, **kw)
        res = plan.run(X)
        assert res.info() == (0, 0, 0)
        single = (rl.slhc3 if algo == "slhc3" else rl.sslhc3)(X, seed=3, cfg=cfg, **kw)
        assert torch.equal(res.piv, single.piv)
        Rh, Rs = res.R.cpu().numpy(), single.R.cpu().numpy()
        assert np.linalg.norm(Rh - Rs) <= 1e-12 * np.linalg.norm(Rs)
        Qh = res.Q.cpu().numpy()
        assert np.linalg.norm(Qh.T @ Qh - np.eye(n)) <= 1e-13 * np.sqrt(n)
        # device errors come back as the first in pipeline order
        Xd = X.clone()
        Xd[:, 5] = 0.0
        assert plan.run(Xd).info()[:2] == (3, 1)  # ERANKDEF, LU
        Xd[777, 3] = float("nan")
        assert plan.run(Xd).info() == (2, 0, 777 * n + 3)  # ENONFINITE, INPUT, element index
        torch.cuda.synchronize()
    if comm is not None:
        comm.close()
