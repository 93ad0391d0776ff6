"""Row-sharded orchestration (paper_2412_06551_b200.dist.DistPlan) on CPU with the gloo
backend and world size 2, stages computed by the oracle (tests/dist_oracle_backend.py).
Checks: pivots bit-identical to the single-process tournament with the same contract
(the tree is global, R#3), R equal to the unsharded oracle's within rounding,
each rank's Q rows equal to the matching rows of the unsharded Q."""
import os
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CASES = [
    # algo, m, n, sketch kwargs, cfg (leaf_rows, arity, panel)
    ("sslhc3", 4096, 24, dict(s1=192, s2=48), (512, 2, 24)),
    ("slhc3", 4096, 40, dict(s=80), (256, 2, 40)),
    ("sslhc3", 8192, 72, dict(s1=576, s2=144), (256, 2, 64)),   # two panels
    # the default contract (128, 8, 16) with shards that are SEVERAL complete subtrees:
    # 16 leaves per rank = 2 subtrees of 8 (K = 2), 3 panels
    ("sslhc3", 4096, 48, dict(s1=384, s2=96), (128, 8, 16)),
    # 3 leaves per rank: no local level at all, every leaf slot is gathered (K = 3)
    ("slhc3", 768, 20, dict(s=40), (128, 8, 16)),
]


def _worker(rank, world, port, algo, m, n, kw, cfgt, out_path):
    sys.path.insert(0, ROOT); sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from dist_oracle_backend import OracleBackend
        from paper_2412_06551_b200._lib import TsluCfg
        from paper_2412_06551_b200.dist import DistPlan
        cfg = TsluCfg(*cfgt)
        mloc = m // world
        X = synth.baseline_matrix(m, n, 10, 5, device="cpu", row0=rank * mloc, rows=mloc)
        plan = DistPlan(algo, m, n, seed=3, cfg=cfg, backend=OracleBackend(cfg), **kw)
        Q, R, piv, infos = plan.run(X)
        np.savez(out_path + f".{rank}.npz", Q=Q.numpy(), R=R.numpy(), piv=piv.numpy(),
                 info=np.array(plan.first_error(infos)))
    finally:
        dist.destroy_process_group()


def _run_dist(world, algo, m, n, kw, cfgt):
    d = tempfile.mkdtemp()
    out = os.path.join(d, "res")
    port = 29500 + (os.getpid() % 1000) + world
    mp.spawn(_worker, args=(world, port, algo, m, n, kw, cfgt, out), nprocs=world, join=True)
    return [np.load(out + f".{r}.npz") for r in range(world)]


@pytest.mark.parametrize("algo,m,n,kw,cfgt", CASES)
def test_two_ranks_match_single_process(ora, algo, m, n, kw, cfgt):
    import synth
    X = synth.baseline_matrix(m, n, 10, 5, device="cpu").numpy()
    b, a, p = cfgt
    ref = ora.slhc3(X, kw["s"], 3, b, a, p) if algo == "slhc3" else ora.sslhc3(X, kw["s1"], kw["s2"], 3, b, a, p)
    res = _run_dist(2, algo, m, n, kw, cfgt)
    for r in res:
        assert tuple(r["info"]) == (0, 0, 0)
        assert np.array_equal(r["piv"], ref.piv)            # global tree -> identical pivots
        assert np.linalg.norm(r["R"] - ref.R) <= 1e-12 * np.linalg.norm(ref.R)
    assert np.array_equal(res[0]["R"], res[1]["R"])          # replicated factors agree bitwise
    Q = np.concatenate([r["Q"] for r in res])
    # Q is determined only to ~kappa * u (kappa = 1e10 here): check it through the gates
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 1e-13 * np.sqrt(n)
    assert np.linalg.norm(Q @ res[0]["R"] - X) <= 1e-14 * n * np.linalg.norm(X)


def test_single_rank_plan_matches_oracle(ora):
    """world = 1 (no process group): the orchestration alone reproduces the monolithic oracle."""
    sys.path.insert(0, HERE)
    import synth
    from dist_oracle_backend import OracleBackend
    from paper_2412_06551_b200._lib import TsluCfg
    from paper_2412_06551_b200.dist import DistPlan
    m, n = 2048, 20
    X = synth.baseline_matrix(m, n, 8, 2, device="cpu")
    cfg = TsluCfg(512, 4, 20)
    plan = DistPlan("sslhc3", m, n, s1=160, s2=40, seed=1, cfg=cfg, backend=OracleBackend(cfg))
    Q, R, piv, infos = plan.run(X)
    ref = ora.sslhc3(X.numpy(), 160, 40, 1, 512, 4, 20)
    assert np.array_equal(piv.numpy(), ref.piv)
    assert np.linalg.norm(R.numpy() - ref.R) <= 1e-13 * np.linalg.norm(ref.R)


def test_shard_contract_and_local_slots():
    """Equal shards of whole leaves are accepted at every GPU count; each rank reduces to
    local_slots complete subtrees (cfg5 = 2^24 rows, 128-row leaves, arity 8: 2^17 leaves)."""
    from paper_2412_06551_b200._lib import TsluCfg, lib
    from paper_2412_06551_b200.dist import check_shard_contract, local_slots
    cfg = TsluCfg(128, 8, 16)
    m = 1 << 24
    for world, k in ((1, 4), (2, 2), (4, 1), (8, 4)):
        check_shard_contract(m, m // world, world, cfg)
        assert local_slots(m // world, cfg) == k
        assert lib().rlhc_tslu_local_slots(m // world, cfg) == k   # the C entry point agrees
    assert local_slots(3 * 128, cfg) == 3
    with pytest.raises(ValueError):
        check_shard_contract(1000, 500, 2, cfg)               # not a multiple of leaf_rows
    with pytest.raises(ValueError):
        check_shard_contract(4096, 1024, 3, cfg)              # unequal shards
    with pytest.raises(ValueError):
        check_shard_contract(4096, 2048, 2, TsluCfg(0, 8, 16))  # invalid contract
