O=gpurun_out
for c in ${CFGL:-cfg2 cfg4a}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$c.csv python tools/prof_cfg.py $c 2 > /dev/null 2>&1
python tools/launches.py $O/l_$c.csv --seq > $O/l_$c.txt
done
