"""Per-kernel warp-stall summary + hottest SASS lines from an ncu --page source csv."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
starts = [i for i, r in enumerate(rows) if r and r[0] == 'Kernel Name'] + [len(rows)]
for si in range(len(starts) - 1):
    blk = rows[starts[si]:starts[si + 1]]
    name = blk[0][1]
    hdr = blk[1]
    ci = {h: i for i, h in enumerate(hdr)}
    if 'Warp Stall Sampling (All Samples)' not in ci:
        continue
    data = [r for r in blk[2:] if len(r) == len(hdr)]
    S = ci['Warp Stall Sampling (All Samples)']
    tot = sum(int(r[S]) for r in data if r[S].isdigit())
    reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    agg = {h: sum(int(r[ci[h]]) for r in data if r[ci[h]].isdigit()) for h in reasons}
    inst = sum(int(r[ci['Instructions Executed']]) for r in data if r[ci['Instructions Executed']].isdigit())
    print(f"=== {name[:90]}\n samples={tot} inst={inst}  " +
          ", ".join(f"{h[6:]}={100*v/max(tot,1):.0f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:6]))
    top = sorted(data, key=lambda r: -int(r[S]) if r[S].isdigit() else 0)[:ntop]
    for r in top:
        rs = sorted([(int(r[ci[h]]), h[6:]) for h in reasons if r[ci[h]].isdigit()], reverse=True)[:2]
        print(f"  {r[S]:>6} x{r[ci['Instructions Executed']]:>8}  {r[ci['Source']].strip()[:58]:58s} {rs}")
