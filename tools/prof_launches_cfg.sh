#!/bin/bash
# ncu launch list (+ DRAM bytes) of one call of a BASELINE config: gpurun_out/l_<cfg>.{csv,txt},
# per-stage traffic into gpurun_out/traffic_<cfg>.json.  Application replay: kernel replay
# would save/restore the 32 GiB buffers of cfg5 around every kernel.
CFG=${1:-cfg5}
O=gpurun_out
timeout ${2:-1200} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --replay-mode application --clock-control none --csv --log-file $O/l_$CFG.csv \
  python tools/prof_cfg.py $CFG 1 > $O/l_$CFG.log 2>&1
echo "ncu rc=$?"
python tools/launches.py $O/l_$CFG.csv > $O/l_$CFG.txt
python tools/traffic.py $O/l_$CFG.csv $CFG $O/traffic_$CFG.json > $O/traffic_$CFG.txt 2>&1
head -40 $O/l_$CFG.txt
