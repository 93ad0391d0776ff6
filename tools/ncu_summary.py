"""Key metrics of one ncu --set full capture (ncu -i rep --page details --csv) -> text summary.

  python tools/ncu_summary.py details.csv "title" > profiles/<name>.txt
"""
import csv
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "One or More Eligible",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
H = {h: i for i, h in enumerate(hdr)}
out = [sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]]
first = next(r for r in rows[1:] if len(r) > H["Metric Value"])
out.append(f"kernel: {first[H['Kernel Name']][:90]}  grid {first[H['Grid Size']]} block {first[H['Block Size']]}")
seen = set()
for r in rows[1:]:
    if len(r) <= H["Metric Value"]:
        continue
    nm = r[H["Metric Name"]]
    if nm in KEEP and nm not in seen:
        seen.add(nm)
        out.append(f"  {r[H['Section Name']][:34]:34s} {nm:36s} {r[H['Metric Value']]:>12s} {r[H['Metric Unit']]}")
print("\n".join(out))
