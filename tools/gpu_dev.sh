#!/bin/bash
# Quick GPU iteration: GPU tests (first failure stops), bench, per-config stage timings.
O=gpurun_out
mkdir -p $O
timeout ${PT_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PT_K:+-k "$PT_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python tools/time_configs.py ${CFGS:-cfg1 cfg2 cfg3 cfg4a cfg4b} > $O/configs.jsonl 2> $O/configs.err
tail -3 $O/pytest_gpu.log; cat $O/bench.json; cat $O/configs.jsonl
