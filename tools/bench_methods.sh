mkdir -p gpurun_out
for m in cholqr2 scholqr3 luc2 rhc auto; do
  timeout 300 python bench.py --method $m --steps 20 --warmup 5 > gpurun_out/bm_$m.json 2> gpurun_out/bm_$m.err
done
for c in cfg3 cfg4a; do for m in cholqr2 scholqr3 luc2 rhc auto; do
  timeout 300 python bench.py --config $c --method $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bm_${c}_$m.json 2> gpurun_out/bm_${c}_$m.err
done; done
