#!/bin/bash
# per-kernel times of the Schur kernels with the LIGHT layout on (every eligible panel) / off
O=gpurun_out
for L in 240 -1; do
  RLHC_SCHUR_LIGHT=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tslw_schur_tma -c 32 --csv --log-file $O/lt2_$L.csv python tools/prof_lu.py 16777216 256 1 > $O/lt2_$L.log 2>&1
done
echo done
