#!/bin/bash
# End-of-session verification on one B200: GPU tests, smoke, bench lines of every config, the
# reference arm, ncu launch list + DRAM bytes per stage for cfg5/cfg3, and a full ncu capture of a
# panel pair's two Schur kernels.  Outputs under gpurun_out/.
O=gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/f_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/f_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/f_smoke.log 2>&1; echo "smoke rc=$?" >> $O/f_smoke.log
timeout 900 python bench.py > $O/f_bench_cfg5.json 2> $O/f_bench_cfg5.err; echo "rc=$?" >> $O/f_bench_cfg5.err
for c in cfg1 cfg2 cfg3 cfg4a cfg4b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/f_bench_$c.json 2> $O/f_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/f_bench_ref_cfg5.json 2> $O/f_bench_ref_cfg5.err
for c in cfg5 cfg3; do
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --replay-mode application --clock-control none --csv --log-file $O/f_l_$c.csv \
    python tools/prof_cfg.py $c 1 > $O/f_l_$c.log 2>&1
  python tools/launches.py $O/f_l_$c.csv > $O/f_l_$c.txt
  python tools/traffic.py $O/f_l_$c.csv $c $O/f_traffic.json > $O/f_traffic_$c.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tslw_schur_tma_kernel -s 12 -c 2 -o $O/f_schur \
   python tools/prof_lu.py 4194304 256 0 > $O/f_schur.log 2>&1
ncu -i $O/f_schur.ncu-rep --page details --csv > $O/f_schur_details.csv 2>&1
ncu -i $O/f_schur.ncu-rep --page raw --csv > $O/f_schur_raw.csv 2>&1
ncu -i $O/f_schur.ncu-rep --page source --csv --print-source sass > $O/f_schur_source.csv 2>&1
rm -f $O/f_schur.ncu-rep
echo done
