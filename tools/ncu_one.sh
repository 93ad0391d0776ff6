#!/bin/bash
# ncu --set full of one kernel (regex $1, skip $2 launches) on a config run: gpurun_out/$3.ncu-rep
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-0} -c 1 -o $O/$3 \
   python tools/prof_cfg.py ${4:-cfg2} 2 > $O/$3.log 2>&1
ncu -i $O/$3.ncu-rep --page details --csv > $O/$3_details.csv 2>&1
ncu -i $O/$3.ncu-rep --page source --csv --print-source sass > $O/$3_source.csv 2>&1
