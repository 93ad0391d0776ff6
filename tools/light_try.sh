#!/bin/bash
# Schur kernel layouts (P4: producer in consumer warp 0 + 4 select warps; LIGHT): parity, LU and
# whole-call timings with the layout on / off, then the in-kernel phase clocks (RLHC_ST_PROF build).
O=gpurun_out
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "getrf or end_to_end or rank_def or edge or graph" > $O/lt_pytest.log 2>&1; echo "rc=$?" >> $O/lt_pytest.log
rm -f $O/lt_lu.txt
for P in default -1 80; do
  for sz in "16777216 256" "1048576 128" "262144 512" "65536 64"; do
    if [ $P = default ]; then unset RLHC_SCHUR_P4; else export RLHC_SCHUR_P4=$P; fi
    echo "P4=$P $sz: $(timeout 300 python tools/prof_lu.py $sz 3 2>&1 | tail -1)" >> $O/lt_lu.txt
  done
done
unset RLHC_SCHUR_P4
echo "P4=default LIGHT=0 16777216 256: $(RLHC_SCHUR_LIGHT=0 timeout 300 python tools/prof_lu.py 16777216 256 3 2>&1 | tail -1)" >> $O/lt_lu.txt
for c in cfg5 cfg3 cfg4b cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/lt_bench_$c.json 2> $O/lt_bench_$c.err
done
RLHC_NVCC_EXTRA="-DRLHC_ST_PROF" python -c "
from paper_2412_06551_b200 import build; build.build(force=True)" > $O/lt_build.log 2>&1
timeout 300 python tools/prof_lu.py 16777216 256 0 > $O/stp_p4.log 2>&1
echo done
