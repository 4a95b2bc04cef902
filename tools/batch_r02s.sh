#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest_r02s.txt 2>&1; echo tests_rc=$?; tail -2 $out/gputest_r02s.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tcf_update_kernel -c 1100 --csv --log-file $out/traffic_r02s_tcf.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo traffic_rc=$?
timeout 1500 python bench.py --steps 2 --warmup 3 > $out/bench_r02s.json 2> $out/bench_r02s.err; echo bench_rc=$?
