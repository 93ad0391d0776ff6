"""Key metrics of a one-kernel ncu --set full report (for profiles/):
python tools/ncu_summary2.py report.ncu-rep"""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
for name, unit, val in zip(h, u, v):
    if name in want:
        print(f"{name:75s} {val:>22s} {unit}")
st = [(name, float(val or 0)) for name, val in zip(h, v) if name.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not name.endswith("not_issued")]
tot = sum(x for _, x in st) or 1.0
print("warp-state samples (share of all):")
for name, x in sorted(st, key=lambda t: -t[1])[:8]:
    print(f"  {name.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f} %")
