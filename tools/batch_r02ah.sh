#!/bin/bash
# bulk-update DRAM traffic at super-column width 12 and 16 (bench config)
out=gpurun_out; mkdir -p $out
for w in 12 16; do
MT_OPTS=6=$w timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tcf_update_kernel -c 1100 --csv --log-file $out/traffic_r02ah_sw$w.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; echo traffic_rc=$?
done
