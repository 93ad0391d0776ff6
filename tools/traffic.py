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
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "").replace("rlhc::", ""))
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1)
        per.setdefault(key, {})[d["Metric Name"]] = v
    return [(k[1], m) for k, m in per.items()]


def split_stages(call):
    """Kernel launches of one call -> stage names (run_algo order)."""
    out = []
    stage = "check_finite"
    seen_tslu = False
    rowsolve_n = 0
    rdiag_n = 0
    for name, m in call:
        base = name.split("<")[0]
        if base in ("status_init_kernel", "check_finite_kernel"):
            stage = "check_finite"
        elif base.startswith(("tslu_", "tslw_", "<unnamed>::tslw_")) or base in ("gather_rows_kernel", "l11_fixup_kernel", "trsm_rows_kernel") \
                and stage in ("check_finite", "tslu"):
            stage = "tslu"
            seen_tslu = True
        elif base in ("fill_i32_kernel", "pivpos_kernel") and seen_tslu:
            stage = "lfactor"
        elif base.startswith(("gauss_", "cs_")):
            stage = "sketch"
        elif base.startswith("hqr"):
            stage = "hqr_y"
        elif base.startswith("chol") or base in ("transpose_kernel", "zero_lower_kernel"):
            stage = {"solve_w_gram1": "chol1", "solve_v_gram2": "chol2"}.get(stage, stage)
        elif base in ("rowsolve_kernel", "subst_ms_kernel", "gemm_update_kernel", "gram_kernel", "gram_reduce_kernel",
                      "gram_part_reduce_kernel", "pivot_rows_kernel"):
            if base in ("rowsolve_kernel", "subst_ms_kernel") or \
                    (base == "gemm_update_kernel" and stage in ("hqr_y", "chol1", "chol2")):
                if stage in ("hqr_y",):
                    stage = "solve_w_gram1"
                elif stage == "chol1":
                    stage = "solve_v_gram2"
                elif stage == "chol2":
                    stage = "solve_q"
                rowsolve_n += 1
        elif base == "rdiag_kernel":
            rdiag_n += 1
        elif base == "trmm_uu_kernel":
            stage = "hqr_y" if stage == "hqr_y" else ("r_finish" if stage == "solve_q" else stage)
        elif base == "status_finish_kernel":
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
    for stage, name, m in split_stages(call):
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
