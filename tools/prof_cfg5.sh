O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_cfg5.csv python tools/prof_cfg.py cfg5 1 > /dev/null 2>&1
python tools/launches.py $O/l_cfg5.csv > $O/l_cfg5.txt
