#!/bin/bash
# Full ncu captures (source-level) of the cfg2 latency-bound kernels.
O=gpurun_out
for k in subst_ms rowsolve_kernel gauss_sketch_kernel hqr_pipe tslw_schur_tma; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o $O/c2_$k \
    python tools/prof_cfg.py cfg2 3 > $O/c2_$k.log 2>&1
  ncu -i $O/c2_$k.ncu-rep --page source --csv --print-source sass > $O/p_c2_${k}_src.csv 2>/dev/null
  ncu -i $O/c2_$k.ncu-rep --page details --csv > $O/p_c2_${k}_details.csv 2>/dev/null
done
ls -la $O | tail -12
