#!/bin/bash
# One measurement session on a GPU box (round 2): bench lines, ncu launch lists with DRAM bytes
# per stage, and full ncu captures of the pass kernels.  Everything lands in gpurun_out/.
O=gpurun_out
set -x
python bench.py > $O/m_bench_cfg5.json 2> $O/m_bench_cfg5.err
for c in cfg1 cfg2 cfg3 cfg4a cfg4b; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/m_bench_$c.json 2> $O/m_bench_$c.err
done
python bench.py --impl reference --steps 3 --warmup 1 > $O/m_bench_ref_cfg5.json 2> $O/m_bench_ref_cfg5.err
for c in cfg2 cfg3 cfg5; do
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --replay-mode application --clock-control none --csv --log-file $O/m_l_$c.csv \
    python tools/prof_cfg.py $c 1 > $O/m_l_$c.log 2>&1
  python tools/launches.py $O/m_l_$c.csv > $O/m_l_$c.txt
  python tools/traffic.py $O/m_l_$c.csv $c $O/m_traffic.json > $O/m_traffic_$c.txt 2>&1
done
for spec in "subst:subst_wide" "gram:syrk_tma" "inv:tri_tma"; do
  what=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -s 1 \
    -o $O/m_ncu_$what python tools/time_pass.py $what 16777216 256 1 > $O/m_ncu_$what.log 2>&1
  ncu -i $O/m_ncu_$what.ncu-rep --page details --csv > $O/m_ncu_${what}_details.csv 2>/dev/null
  ncu -i $O/m_ncu_$what.ncu-rep --page raw --csv > $O/m_ncu_${what}_raw.csv 2>/dev/null
done
python tools/pcie_bw.py 16 > $O/m_pcie.txt 2>&1
echo done
