#!/usr/bin/env python
"""bench.py -- SLHC3 / SSLHC3 (arXiv 2412.06551) fp64 QR on B200: time and HBM GB/s
against the roofline (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]

One JSON line on rank 0.  A step = one full SLHC3/SSLHC3 call (every stage of
SURVEY.md 8(a)) on the configuration's synthetic X, resident in HBM.  The default workload
is BASELINE.json's headline: cfg5, SSLHC3 on m = 2^24, n = 256 (the metric is quoted "at
1/2/4/8 B200" on it; it fits one B200).  `value` is the algorithmic HBM throughput of the
whole job: the bytes of the 8 required passes over m x n data (8 * 8 m n bytes, DESIGN.md
section 6) per second of device time (max over ranks).  X (32 GiB at cfg5) is far larger
than L2; L2 is also flushed between timed steps (a 512 MiB write, outside the timed events).
N > 1 runs the row-sharded algorithm (paper_2412_06551_b200.dist) with NCCL: by default
strong scaling of the config's m (the north star: cfg5 at 1/2/4/8 GPUs); --weak gives every
rank the config's m rows.  Every arm runs the same pivot contract, restated below
(TSLU_CONTRACT), on the GPU and in the oracle.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAK_FP64_DMMA_TFLOPS = 37.08  # measured by tools/probe/probe.cu (profiles/r01_probe_fp64_hbm.txt)
# scalar FP64 FMA (DFMA) peak: measured 36.86 TF/s (same probe); from unit counts
# 148 SMs x 64 FP64 lanes x 2 flop x 1.965 GHz = 37.2 TF/s.  The FP64 pipe
# issues 148 x 64 x 1.965e9 = 18.6e12 lane-operations per second; a DMUL or DADD is one of them
# (a DFMA too, for two flops), so the oracle-order substitution (a rounded product, then a
# rounded difference per term) is bound by PEAK_FP64_OPS, not by the FMA flop rate.
PEAK_FP64_ALU_TFLOPS = 36.86
PEAK_FP64_OPS_T = PEAK_FP64_ALU_TFLOPS / 2  # 1e12 FP64 pipe operations per second
ALU_STAGES = {"tslu"}  # scalar-FMA stages (GEPP select / elimination), not tensor-core work
OPS_STAGES = {"solve_w"}  # scalar DMUL + DADD (n > 64; subst_wide_tma_kernel), counted in pipe ops


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def stage_model(cfg: synth.Config) -> dict:
    """Algorithmic bytes and work per stage: (bytes, flops) -- for
    solve_w at n > 64 the work is FP64 pipe operations (n(n-1) products and differences + n
    divisions per row), for the others flops."""
    m, n = cfg.m, cfg.n
    M = 8.0 * m * n
    tri = m * n * (n + 1.0)  # triangular row product / Gram upper half: flops
    srows = cfg.s if cfg.algo == "slhc3" else cfg.s1
    sk_flops = 2.0 * cfg.s * m * n if cfg.algo == "slhc3" else m * n + 2.0 * cfg.s2 * cfg.s1 * n
    fused = n <= 64  # the solve kernels fuse their Gram (the gram stages are empty)
    return {
        # tslu: the warp tournament reads X and writes L (the L factor is its by-product,
        # the lfactor stage is empty); m n^2 flop of elimination + the panels' Schur updates
        "check_finite": (M, 0.0), "tslu": (2 * M, m * n * n * 1.0), "lfactor": (2 * M, m * n * n * 1.0),
        "sketch": (M + 8.0 * srows * n, sk_flops), "hqr_y": (0.0, 2.0 * srows * n * n),
        "solve_w": (2 * M, (m * n * n + tri) if fused else m * n * n * 1.0), "gram1": (M, tri),
        "chol1": (0.0, n ** 3 / 3.0),
        "solve_v": (2 * M, (m * n * n + tri) if fused else tri), "gram2": (M, tri),
        "chol2": (0.0, n ** 3 / 3.0),
        "solve_q": (2 * M, m * n * n * 1.0 if fused else tri), "r_finish": (0.0, 2.0 * n ** 3 / 3),
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


_CHECK: dict = {}


def check_result(X, res, n: int) -> dict:
    """Gates on the LAST timed step's output, outside every timed region (verification only:
    plain torch fp64, chunked): ||Q^T Q - I||_F <= 1e-13 sqrt(n) and, on the first and last 65536
    rows, ||Q R - X||_F / ||X||_F <= 1e-14 n (the tests' gates); diag(R) > 0.  A step that timed
    garbage fails the bench instead of printing a number."""
    Q, R = res.Q, res.R
    m = Q.shape[0]
    G = torch.zeros(n, n, dtype=torch.float64, device=Q.device)
    step = 1 << 20
    for i in range(0, m, step):
        G.addmm_(Q[i:i + step].T, Q[i:i + step])
    orth = float(torch.linalg.norm(G - torch.eye(n, dtype=torch.float64, device=Q.device)))
    num = den = 0.0
    rows = sorted({0, max(0, m - 65536)})
    for i in rows:
        d = Q[i:i + 65536] @ R - X[i:i + 65536]
        num += float((d * d).sum())
        den += float((X[i:i + 65536] ** 2).sum())
    resid = (num / max(den, 1e-300)) ** 0.5
    diag_pos = bool((torch.diagonal(R) > 0).all())
    out = {"orth_fro": orth, "resid_sample": resid, "diag_R_positive": diag_pos,
           "gates": {"orth_fro": 1e-13 * n ** 0.5, "resid_sample": 1e-14 * n}}
    if not (orth <= out["gates"]["orth_fro"] and resid <= out["gates"]["resid_sample"] and diag_pos):
        raise RuntimeError(f"timed step's result fails its gates: {out}")
    return out


def run_ours(args, cfg: synth.Config, rank: int, world: int):
    import paper_2412_06551_b200 as rl
    from paper_2412_06551_b200 import _lib
    # RLHC_BENCH_FUNCTIONAL=1: every rank on cuda:0 with gloo -- a functional check of the
    # N > 1 code path on a one-GPU box, never a timing
    functional = os.environ.get("RLHC_BENCH_FUNCTIONAL") == "1"
    dev = torch.device("cuda", 0 if functional else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    tcfg = None
    if world > 1:
        from paper_2412_06551_b200 import dist as rdist
        X, plan = rdist.setup_bench(cfg, rank, world, dev, strong=not args.weak, use_c=not functional,
                                    contract=_default_cfg_tuple(cfg))
        run = lambda: plan.run(X)  # noqa: E731
    else:
        X = synth.config_matrix(cfg, device=dev)
        if args.method in METHOD_PASSES:
            s1, s2 = _rhc_sizes(cfg)
            plan = rl.MethodPlan(args.method, cfg.m, cfg.n, s1=s1, s2=s2, seed=cfg.seed, cfg=_default_cfg_tuple(cfg),
                                 device=dev)
        else:
            # the restated contract (TSLU_CONTRACT); --pivot gepp: one leaf = exact GEPP
            tcfg = (cfg.m, 2, min(16, cfg.n)) if args.pivot == "gepp" else _default_cfg_tuple(cfg)
            plan = rl.Plan(cfg.algo, cfg.m, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, seed=cfg.seed, cfg=tcfg, device=dev)
        run = lambda: plan.run(X)  # noqa: E731
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        res = run()
    torch.cuda.synchronize(dev)
    code = res.info()
    if code[0] != 0:
        raise RuntimeError(f"warm-up run failed: info={code}")
    # stage breakdown and kernels per call from direct calls (untimed)
    _lib.lib().rlhc_stage_timing(1)
    _lib.stage_times()  # drain
    l0 = _lib.lib().rlhc_launch_count()
    for _ in range(3):
        flush.zero_()
        res = run()
    torch.cuda.synchronize(dev)
    per_call = (_lib.lib().rlhc_launch_count() - l0) // 3
    stages = _lib.stage_times()
    _lib.lib().rlhc_stage_timing(0)
    # timed steps: one CUDA graph launch per step (rlhc_graph_*, the whole call captured once)
    use_graph = args.graph and world == 1 and isinstance(plan, rl.Plan)
    if use_graph:
        plan.capture(X)
        run = plan.replay
        for _ in range(args.warmup):
            res = run()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush (outside the timed events)
            evs[k][0].record(stream)
            res = run()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = per_call * args.steps
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    code = res.info()
    if code[0] != 0:
        raise RuntimeError(f"timed run failed: info={code}")
    if world == 1:
        _CHECK.update(check_result(X, res, cfg.n))

    # ---- end to end through the public API with host buffers: every step copies this
    # rank's rows of X from pinned host memory and reads Q (its rows) and R back; device
    # time, max over ranks.  The device-resident buffers of the timed part are released
    # first (cfg5: X, Q are 32 GiB each; the host pipeline double-buffers both).
    m_rows = X.shape[0]
    Xh = torch.empty(m_rows, cfg.n, dtype=torch.float64).pin_memory()
    Xh.copy_(X)
    Qh = torch.empty(m_rows, cfg.n, dtype=torch.float64).pin_memory()
    Rh = torch.empty(cfg.n, cfg.n, dtype=torch.float64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    big = 8 * m_rows * cfg.n > (4 << 30)
    # K problems streamed like the device-side K steps (each cfg5 step moves 64 GiB over PCIe:
    # ~0.8 s at the measured 91 GB/s duplex rate, tools/pcie_bw.py; the pipeline's fill and
    # drain -- one H2D before the first solve, one D2H after the last -- amortise over K)
    e2e_steps = args.steps
    e2e_warm = 1 if big else args.warmup
    e2e = {"unit": "GB/s", "h2d_bytes_per_step": 8 * m_rows * cfg.n,
           "d2h_bytes_per_step": 8 * (m_rows * cfg.n + cfg.n * cfg.n), "per": "rank", "steps": e2e_steps}
    if world == 1 and isinstance(plan, rl.Plan):
        del X, plan, run, res
        torch.cuda.empty_cache()
        # K problems through rlhc_host_pipeline (host X -> host Q, R; the H2D copy of step k+1
        # and the D2H copy of step k-1 overlap step k's computation); the serial latency of
        # one call (copy in, compute, copy out) from a pipeline of one problem
        hp = rl.HostPipeline(cfg.algo, m_rows, cfg.n, s=cfg.s, s1=cfg.s1, s2=cfg.s2, cfg=tcfg, device=dev)
        hp.run([Xh] * e2e_warm, [cfg.seed] * e2e_warm, [Qh] * e2e_warm, [Rh] * e2e_warm)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        hp.run([Xh], [cfg.seed], [Qh], [Rh])
        e1.record(stream)
        e1.synchronize()
        e2e["latency_ms_per_call"] = e0.elapsed_time(e1)
        e0.record(stream)
        hp.run([Xh] * e2e_steps, [cfg.seed] * e2e_steps, [Qh] * e2e_steps, [Rh] * e2e_steps)
        e1.record(stream)
        e1.synchronize()
        bad = [c for c in hp.infos() if c[0] != 0]
        if bad:
            raise RuntimeError(f"host pipeline run failed: {bad[0]}")
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        e2e["api"] = "rlhc_host_pipeline (K steps streamed; copies overlap compute)"
        del hp
        X = None
    else:
        Xd = torch.empty_like(X)
        tot = 0.0
        for k in range(e2e_warm + e2e_steps):
            flush.zero_()
            if world > 1:
                torch.distributed.barrier()
            e0.record(stream)
            Xd.copy_(Xh, non_blocking=True)
            r2 = plan.run(Xd)
            Qh.copy_(r2.Q, non_blocking=True)
            Rh.copy_(r2.R, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if k >= e2e_warm:
                tot += e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([tot], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            tot = float(t.item())
        e2e_ms = tot / e2e_steps
        e2e["api"] = ("rlhc_slhc3_dist / rlhc_sslhc3_dist per step (copies serial)" if world > 1
                      else "MethodPlan.run per step (copies serial)")
    e2e["ms_per_step"] = e2e_ms
    return ms, stages, launches, clk.summary(), e2e, Xh


def roofline(cfg: synth.Config, stages: dict, world: int, step_ms: float = 0.0, m_local: int = 0, passes: int = 8):
    calls = max(stages.get("calls", 1), 1)
    model = stage_model(cfg)
    hbm, hbm_src = _peaks()
    if not any(v for k, v in stages.items() if k != "calls"):
        # N > 1 and the comparison algorithms have no stage markers: the whole step of one
        # rank against its HBM roof (the algorithmic passes over its rows)
        byts = passes * 8.0 * m_local * cfg.n
        ach = byts / (step_ms * 1e-3) / 1e9
        return {"kernel": "whole step (per rank)", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "peak_source": hbm_src, "ms": step_ms}
    best = None
    for name, (byts, flops) in model.items():
        t = stages.get(name, 0.0) / calls * 1e-3
        if t <= 0:
            continue
        # the dominant KERNEL: at n > 64 every stage but tslu (16 tournaments, 15 Schur kernels,
        # U rows, ...) is one kernel launch (solve_w = subst_wide, gram = gram_kernel, ...)
        if name == "tslu" and cfg.n > 64:
            continue
        if best is None or t > best[1]:
            best = (name, t, byts, flops)
    name, t, byts, flops = best
    t_hbm, t_fp = byts / (hbm * 1e9), flops / (PEAK_FP64_DMMA_TFLOPS * 1e12)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = prof.get(f"{cfg.name}:{name}")
    except Exception:
        pass
    if name in OPS_STAGES and cfg.n > 64:
        ach = flops / t / 1e12
        return {"kernel": "subst_wide_tma_kernel (" + name + ")", "bound": "alu", "achieved": ach, "peak": PEAK_FP64_OPS_T,
                "unit": "T FP64-pipe ops/s", "frac": ach / PEAK_FP64_OPS_T, "traffic": traffic,
                "peak_source": "the scalar DFMA instruction rate measured on this pool (36.86 TF/s = 18.43 T "
                               "DFMA/s, profiles/r01_probe_fp64_hbm.txt); a DMUL or a DADD costs the FP64 "
                               "pipe what a DFMA does (tools/probe/pdmuladd.cu, profiles/r02_probe_dmul_dadd.txt)",
                "ms": t * 1e3, "note": "oracle-order substitution: a rounded product and a rounded difference "
                                       "per term (DESIGN.md R#O9), no FMA"}
    if name in ALU_STAGES:
        ach = flops / t / 1e12
        return {"kernel": name, "bound": "alu", "achieved": ach, "peak": PEAK_FP64_ALU_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / PEAK_FP64_ALU_TFLOPS, "traffic": traffic,
                "peak_source": "scalar fp64 FMA measured on this pool (profiles/r01_probe_fp64_hbm.txt)",
                "ms": t * 1e3, "note": "latency-bound tournament (levels x n sequential GEPP steps)"}
    if t_fp >= t_hbm:
        ach = flops / t / 1e12
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": PEAK_FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / PEAK_FP64_DMMA_TFLOPS, "traffic": traffic,
                "peak_source": "fp64 DMMA measured on this pool (profiles/r01_probe_fp64_hbm.txt)",
                "ms": t * 1e3}
    ach = byts / t / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "traffic": traffic, "peak_source": hbm_src, "ms": t * 1e3}


def sample_rows(cfg: synth.Config) -> int:
    """Rows of the oracle's bounded sample: the whole X up to 2^24 entries (cfg1, cfg2), else
    the first rows of X holding 2^24 entries (cfg3: 131072 rows, cfg4: 32768, cfg5: 65536;
    a few seconds of oracle work on 16 host cores).  Never fewer than the sketch rows
    (s <= m, s1 <= m)."""
    if cfg.m * cfg.n <= (1 << 24):
        return cfg.m
    return min(cfg.m, max((1 << 24) // cfg.n, cfg.s, cfg.s1, 1))


def cpu_baseline(cfg: synth.Config, Xh: torch.Tensor | None, budget_s: float = 8.0, method: str = "auto",
                 max_reps: int = 20, warm: int = 0):
    """The oracle (oracle/, plain C, all host cores) on a bounded sample of the workload: the
    first sample_rows(cfg) rows of the same X bytes (the whole X for cfg1-cfg3), the same
    sketch sizes, seed and pivot contract.  value = the metric's bytes for the sample / time."""
    import oracle
    oracle.build()
    ms_ = sample_rows(cfg)
    if Xh is None:
        Xh = synth.baseline_matrix(cfg.m, cfg.n, cfg.kappa_exp, cfg.seed, cfg.colscale,
                                   device="cuda" if torch.cuda.is_available() else "cpu", rows=ms_).cpu()
    Xs = Xh[:ms_].numpy()
    b, a, p = _default_cfg_tuple(cfg)

    def one():
        if method in METHOD_PASSES:
            s1, s2 = _rhc_sizes(cfg)
            {"cholqr2": lambda: oracle.cholqr2(Xs), "scholqr3": lambda: oracle.scholqr3(Xs),
             "luc2": lambda: oracle.luc2(Xs, b, a, p), "rhc": lambda: oracle.rhc(Xs, s1, s2, cfg.seed)}[method]()
        elif cfg.algo == "slhc3":
            oracle.slhc3(Xs, cfg.s, cfg.seed, b, a, p)
        else:
            oracle.sslhc3(Xs, cfg.s1, cfg.s2, cfg.seed, b, a, p)

    for _ in range(warm):
        one()
    reps, t0 = 0, time.perf_counter()
    while True:
        one()
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= max_reps:
            break
    per = el / reps
    what = f"full {cfg.name} ({cfg.m}x{cfg.n})" if ms_ == cfg.m else \
        f"first {ms_} of {cfg.m} rows of {cfg.name}'s X ({ms_}x{cfg.n}, same sketch sizes, seed, contract {b, a, p})"
    return {"value": _passes(method) * 8.0 * ms_ * cfg.n / per / 1e9, "unit": "GB/s", "cores": oracle.num_threads(),
            "kind": "oracle", "sample": f"{what} x{reps}", "s_per_step": per}


# the paper's comparison algorithms, 1 GPU: algorithmic passes over m x n
# data in the paper's order: CholeskyQR = Gram (1 read) + substitution
# (read + write) = 3; LUC2 = LU (read X, write L) + Gram(L) + W = X Y^-1 + CholeskyQR(W) = 8;
# RHC = sketch (1) + W = X Y^-1 (2) + CholeskyQR(W) (3) = 6
METHOD_PASSES = {"cholqr2": 6, "scholqr3": 9, "luc2": 8, "rhc": 6}


def _passes(method: str) -> int:
    return METHOD_PASSES.get(method, 8)


def _rhc_sizes(cfg):
    # RHC's CountSketch / Gaussian sizes: the SSLHC3 ones (s1 = 8n, s2 = 2n, BASELINE.json)
    return min(cfg.m, cfg.s1 or 8 * cfg.n), cfg.s2 or 2 * cfg.n


def _default_cfg_tuple(cfg):
    """The tournament pivot contract every arm runs (R#3), restated here rather than
    read from the product library: 128-row leaves, 8-ary nodes, 16-column panels (CALU);
    both the GPU and the oracle are handed exactly this tuple."""
    return TSLU_CONTRACT[0], TSLU_CONTRACT[1], min(cfg.n, TSLU_CONTRACT[2])


TSLU_CONTRACT = (128, 8, 16)  # (leaf_rows, arity, panel)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", help="BASELINE.json config (cfg5 = the headline)")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: every rank holds the config's m rows (default: strong scaling, the config's m "
                         "split over the ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="time the call as one CUDA graph launch per step (default, N = 1)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--pivot", default="tournament", choices=["tournament", "gepp"],
                    help="pivot contract: the default tournament (CALU) or exact GEPP (one leaf, SURVEY 8(f) NEXT-2)")
    ap.add_argument("--kappa-exp", type=int, default=None,
                    help="override the config's kappa = 1e<k> (default for --method cholqr2: min(k, 6), "
                         "CholeskyQR2 breaks down once kappa^2 u > 1, P:34)")
    ap.add_argument("--method", default="auto", choices=["auto"] + sorted(METHOD_PASSES),
                    help="auto: the config's SLHC3/SSLHC3; else one of the paper's comparison algorithms "
                         "(1 GPU) on the same X")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    cfg = synth.CONFIGS[args.config]
    if args.kappa_exp is not None:
        cfg = dataclasses.replace(cfg, kappa_exp=args.kappa_exp)
    elif args.method == "cholqr2" and cfg.kappa_exp > 6:
        cfg = dataclasses.replace(cfg, kappa_exp=6)
    strong = world > 1 and not args.weak
    m_global = cfg.m if (strong or world == 1) else cfg.m * world
    if world > 1 and not torch.distributed.is_initialized():
        functional = os.environ.get("RLHC_BENCH_FUNCTIONAL") == "1"
        torch.distributed.init_process_group("nccl" if args.impl == "ours" and not functional else "gloo")
    if args.method != "auto" and world > 1:
        raise SystemExit("--method: the comparison algorithms run on 1 GPU")
    algo = cfg.algo if args.method == "auto" else args.method
    passes = _passes(args.method)
    s1m, s2m = _rhc_sizes(cfg)
    sizes = (f"s={cfg.s}" if algo == "slhc3" else f"s1={cfg.s1} s2={cfg.s2}" if algo == "sslhc3"
             else f"s1={s1m} s2={s2m}" if algo == "rhc" else "")
    workload = (f"{cfg.name}: {algo.upper()} m={m_global} n={cfg.n}" + (" " + sizes if sizes else "")
                + f" kappa=1e{cfg.kappa_exp}{' colscale' if cfg.colscale else ''} seed={cfg.seed}")
    contract = (cfg.m, 2, min(16, cfg.n)) if args.pivot == "gepp" else _default_cfg_tuple(cfg)
    base = {"metric": f"{algo.upper()} fp64 QR algorithmic HBM throughput ({passes} passes of m x n)",
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "m": m_global, "n": cfg.n, "s": cfg.s, "s1": cfg.s1, "s2": cfg.s2,
                       "kappa": f"1e{cfg.kappa_exp}",
                       "tslu_contract": {"leaf_rows": contract[0], "arity": contract[1], "panel": contract[2]},
                       "l2": (f"X ({8 * m_global * cfg.n / 2**30:.1f} GiB) larger than L2; also flushed between "
                              "steps (512 MiB write)") if 8 * m_global * cfg.n > (256 << 20)
                       else "flushed between steps (512 MiB write)",
                       "rows_per_gpu": m_global // world,
                       "parallelism": f"row-sharded x{world} (NCCL)" if world > 1 else "1 GPU",
                       "launch": ("one CUDA graph per step (rlhc_graph_*)" if args.graph and world == 1
                                  and args.method in ("auto", "slhc3", "sslhc3") else "stream launches")}}
    if args.impl == "reference":
        if rank != 0:
            return
        # the oracle as it stands, each step one bounded sample of the workload (sample_rows)
        cb = cpu_baseline(cfg, None, budget_s=1e9, method=args.method, max_reps=args.steps, warm=args.warmup)
        line = dict(base, impl="reference", value=cb["value"], ms_per_step=cb["s_per_step"] * 1e3,
                    cpu_baseline=cb, e2e={"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}, n_gpus=0)
        print(json.dumps(line), flush=True)
        return
    ms, stages, launches, clocks, e2e, Xh = run_ours(args, cfg, rank, world)
    if rank != 0:
        return
    per_step = ms / args.steps
    value = passes * 8.0 * m_global * cfg.n / (per_step * 1e-3) / 1e9  # whole job, all ranks
    e2e["value"] = passes * 8.0 * m_global * cfg.n / (e2e.pop("ms_per_step") * 1e-3) / 1e9
    e2e["ms_per_step"] = passes * 8.0 * m_global * cfg.n / e2e["value"] / 1e6
    line = dict(base, value=value, ms_per_step=per_step, gpu_launches=launches, clocks=clocks,
                roofline=roofline(cfg, stages, world, per_step, m_global // world, passes), e2e=e2e,
                stages_ms={k: v / max(stages.get("calls", 1), 1) for k, v in stages.items() if k != "calls" and v})
    if _CHECK:
        line["check"] = dict(_CHECK)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, Xh, method=args.method)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
