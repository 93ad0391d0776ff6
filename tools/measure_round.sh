#!/bin/bash
# One measurement session on a GPU box (round 2): bench lines, ncu launch lists with DRAM bytes
# per stage, and one full ncu capture of the dominant kernel.  Everything lands in gpurun_out/.
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
timeout 900 ncu --set full --import-source on --clock-control none -k regex:subst_wide -c 1 -s 1 \
  -o $O/m_ncu_subst_wide python tools/prof_trmm.py subst 1048576 256 > $O/m_ncu_subst_wide.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ts_gemm -c 1 -s 1 \
  -o $O/m_ncu_ts_gemm python tools/prof_trmm.py inv 4194304 256 > $O/m_ncu_ts_gemm.log 2>&1
echo done
