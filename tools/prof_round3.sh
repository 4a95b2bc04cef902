#!/bin/bash
tag=${1:-r01d}
out=gpurun_out; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2_update_kernel -s 30 -c 2 \
  -o $out/full_${tag}_tc2_update_kernel python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > $out/ncu_${tag}_tc2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:"tc2_update_kernel|dmma_tma_update_kernel|gen_kernel" -c 1500 --csv \
  --log-file $out/traffic_${tag}_n262144.csv python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > $out/ncu_${tag}_traffic.log 2>&1
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo bench_rc=$?
echo done
