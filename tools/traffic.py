"""Per-stage DRAM traffic of one SLHC3/SSLHC3 call from an ncu CSV with the metrics
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum (one row per launch).

  python tools/traffic.py <ncu.csv> <cfg name> [profiles/traffic.json]

The last complete call (status_init ... status_finish) is split into the stages of
rlhc.cu's run_algo by launch order; bench.py reports the dominant stage's bytes per call as
roofline.traffic (read + write, to compare with the stage's algorithmic bytes).
"""
import csv
import json
import sys
from collections import OrderedDict

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "").replace("rlhc::", "")
               .replace("<unnamed>::", ""))
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1)
        per.setdefault(key, {})[d["Metric Name"]] = v
    return [(k[1], m) for k, m in per.items()]


def _base(name):
    """Kernel base name: namespaces and template arguments stripped."""
    b = name.replace("<unnamed>::", "").replace("rlhc::", "").replace("void ", "")
    return b.split("<")[0].split("::")[-1]


def split_stages(call, n):
    """Kernel launches of one call -> stage names (run_algo order, rlhc.cu kStageNames).
    After HouseholderQR each CholeskyQR pass starts with a recognisable kernel: the W solve
    (subst_ms / subst_wide), tri_inv for V and Q when n > 64 (rowsolve when n <= 64; the
    blocked Cholesky of n > 128 also runs rowsolve / gemm_sub inside its stage), the Gram
    (gram_kernel or syrk_tma_kernel), the Cholesky (chol_*), the final trmm_uu."""
    out = []
    stage = "check_finite"
    post = False
    for name, m in call:
        b = _base(name)
        pass_start = b == "tri_inv_kernel" if n > 64 else b == "rowsolve_kernel"
        if not post:
            if b in ("status_init_kernel", "check_finite_kernel"):
                stage = "check_finite"
            elif b.startswith(("tslu_", "tslw_", "tslg_", "gather_rows", "l11_fixup", "trsm_rows", "pivpos",
                               "fill_i32")) or (b in ("ts_gemm_kernel", "pack_b_kernel") and stage == "tslu"):
                stage = "tslu"
            elif b.startswith(("gauss_", "cs_", "omega_gen")):
                stage = "sketch"
            elif b.startswith("hqr") or (stage == "hqr_y" and b in ("trmm_uu_kernel", "rdiag_kernel")):
                stage = "hqr_y"
            elif stage == "hqr_y" and b in ("subst_ms_kernel", "subst_wide_kernel", "subst_wide_tma_kernel", "rowsolve_kernel",
                                            "gemm_sub_kernel"):
                post = True
                stage = "solve_w"
        else:
            if b in ("gram_kernel", "syrk_tma_kernel"):
                stage = {"solve_w": "gram1", "solve_v": "gram2"}.get(stage, stage)
            elif b.startswith("chol_"):
                stage = {"solve_w": "chol1", "gram1": "chol1", "solve_v": "chol2", "gram2": "chol2"}.get(stage, stage)
            elif pass_start:
                stage = {"chol1": "solve_v", "chol2": "solve_q"}.get(stage, stage)
            elif b == "trmm_uu_kernel" and stage == "solve_q":
                stage = "r_finish"
        out.append((stage, name, m))
    return out


def main():
    path, cfg = sys.argv[1], sys.argv[2]
    dst = sys.argv[3] if len(sys.argv) > 3 else None
    ls = launches(path)
    calls, cur = [], []
    for name, m in ls:
        if name.startswith("status_init") and cur:
            calls.append(cur)
            cur = []
        cur.append((name, m))
    calls.append(cur)
    call = calls[-1]
    agg = OrderedDict()
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    for stage, name, m in split_stages(call, synth.CONFIGS[cfg].n):
        a = agg.setdefault(stage, {"us": 0.0, "dram_bytes": 0.0, "kernels": 0})
        a["us"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["kernels"] += 1
    for k, a in agg.items():
        print(f"{k:15s} {a['kernels']:3d} kernels {a['us']:9.1f} us  dram {a['dram_bytes'] / 1e6:9.2f} MB")
    if dst:
        try:
            cur = json.load(open(dst))
        except Exception:
            cur = {}
        for k, a in agg.items():
            cur[f"{cfg}:{k}"] = a["dram_bytes"]
        json.dump(cur, open(dst, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
