"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel times of the last call."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            if d['Metric Unit'] == 'usecond':
                v *= 1000
            elif d['Metric Unit'] == 'msecond':
                v *= 1e6
            out.append((d['Kernel Name'].split('(')[0].replace('void ', '').replace('rlhc::', ''), v))
# split calls at status_init
calls, cur = [], []
for k, v in out:
    if k.startswith('status_init') and cur:
        calls.append(cur); cur = []
    cur.append((k, v))
calls.append(cur)
last = calls[-1]
tot = sum(v for _, v in last)
agg = OrderedDict()
for k, v in last:
    agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += v
print(f"calls={len(calls)} kernels/call={len(last)} total={tot/1000:.1f} us")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {v/1000:9.1f} us  {100*v/tot:5.1f}%  x{c:<3d} {k}")
if len(sys.argv) > 2 and sys.argv[2] == "--seq":
    for k, v in last:
        print(f"  {v/1000:9.2f} us  {k}")
