#!/bin/bash
# One GPU session: build check, GPU tests, bench, per-config stage timings, ncu launch list,
# per-launch DRAM traffic, one full capture of the top kernel.  Outputs under gpurun_out/.
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python tools/time_configs.py ${CFGS:-cfg1 cfg2 cfg3 cfg4a cfg4b cfg5} > $O/configs.jsonl 2> $O/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/traffic.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${TOPK:-tslw_tree_kernel} -s ${TOPS:-2} -c 1 -o $O/top \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
ls -la $O
python tools/traffic.py $O/traffic.csv cfg2 $O/traffic.json > $O/traffic_stages.txt 2>&1
ncu -i $O/top.ncu-rep --page details --csv > $O/top_details.csv 2>&1
python tools/ncu_summary.py $O/top_details.csv "ncu --set full --clock-control none -k regex:${TOPK:-tslw_tree_kernel} (bench.py cfg2)" > $O/top_summary.txt 2>&1
