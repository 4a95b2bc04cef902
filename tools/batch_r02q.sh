#!/bin/bash
# ncu evidence for the final tcf layout: DRAM traffic per bulk launch at the bench config,
# one full capture of a mid-factorization bulk launch (N=131072, step 40, no co-scheduling)
out=gpurun_out; mkdir -p $out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tcf_update_kernel -c 1100 --csv --log-file $out/traffic_r02q_tcf.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo traffic_rc=$?
MT_OPTS=10=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcf_update_kernel -s 81 -c 1 \
  -o $out/full_r02q_tcf python tools/prof_eval.py --n 131072 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo full_rc=$?
