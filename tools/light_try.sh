#!/bin/bash
# Schur kernel experiment: parity subset, LU timings, whole-call bench, then the phase clocks.
O=gpurun_out
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "getrf or end_to_end or rank_def or edge or graph" > $O/lt_pytest.log 2>&1; echo "rc=$?" >> $O/lt_pytest.log
grep -q "rc=0" $O/lt_pytest.log || exit 1
rm -f $O/lt_lu.txt
for sz in "16777216 256" "1048576 128" "262144 512" "65536 64"; do
  echo "$sz: $(timeout 300 python tools/prof_lu.py $sz 3 2>&1 | tail -1)" >> $O/lt_lu.txt
done
for c in cfg5 cfg3 cfg4b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/lt_bench_$c.json 2> $O/lt_bench_$c.err
done
RLHC_NVCC_EXTRA="-DRLHC_ST_PROF" python -c "
from paper_2412_06551_b200 import build; build.build(force=True)" > $O/lt_build.log 2>&1
timeout 300 python tools/prof_lu.py 16777216 256 0 > $O/stp_lt.log 2>&1
echo done
