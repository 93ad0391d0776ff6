#!/bin/bash
# Full ncu captures (source-level) of the three streaming-pass kernels at cfg5 size.
O=gpurun_out
M=${M:-16777216}
N=${N:-256}
for spec in "gram:gram_kernel" "subst:subst_wide_tma" "inv:ts_gemm"; do
  what=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o $O/p_$what \
    python tools/time_pass.py $what $M $N 1 > $O/p_$what.log 2>&1
  ncu -i $O/p_$what.ncu-rep --page source --csv --print-source sass > $O/p_${what}_src.csv 2>/dev/null
  ncu -i $O/p_$what.ncu-rep --page details --csv > $O/p_${what}_details.csv 2>/dev/null
  ncu -i $O/p_$what.ncu-rep --page raw --csv > $O/p_${what}_raw.csv 2>/dev/null
done
ls -la $O
