#!/bin/bash
# N = 2 code path of bench.py on a one-GPU box: both ranks on cuda:0 over gloo (a functional
# check of the row-sharded path through torch.distributed, never a timing)
O=gpurun_out
RLHC_BENCH_FUNCTIONAL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/bench_n2_functional.json 2> $O/bench_n2_functional.err
echo "rc=$?" >> $O/bench_n2_functional.err
