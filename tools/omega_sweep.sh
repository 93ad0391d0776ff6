#!/bin/bash
# Omega side-stream sweep: store on/off x generator CTAs per SM on cfg2 / cfg4a / cfg3.
O=gpurun_out; mkdir -p $O; : > $O/omega_sweep.jsonl
for st in 0 1; do for c in 1 2 4 8; do
  [ $st = 0 ] && [ $c != 2 ] && continue
  RLHC_OMEGA_STORE=$st RLHC_OMEGA_CTAS=$c timeout 600 python tools/time_configs.py ${CFGS:-cfg2 cfg4a cfg3} 2>>$O/omega_sweep.err \
    | sed "s/^{/{\"store\": $st, \"ctas\": $c, /" >> $O/omega_sweep.jsonl
done; done
cat $O/omega_sweep.jsonl | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); st=r['stages_ms']; print(r['store'],r['ctas'],r['cfg'],round(r['ms'],3),'tslu',st['tslu'],'sketch',st['sketch'])"
