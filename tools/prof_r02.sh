#!/bin/bash
# Round-2 measurement pass on one B200: bench line, ncu launch list of the bench
# command, DRAM traffic of the bulk update at the bench config, one full ncu
# capture of the bulk update kernel.
out=gpurun_out; mkdir -p $out
tag=${1:-r02}
timeout 1200 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo bench_rc=$?
tail -c 600 $out/bench_$tag.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -c 5300 --csv --log-file $out/launches_${tag}_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dp --no-e2e > $out/bench_under_ncu_$tag.log 2>&1
echo launches_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tcf_update_kernel -c 1100 --csv --log-file $out/traffic_${tag}_tcf.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo traffic_rc=$?
MT_OPTS=10=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcf_update_kernel -s 81 -c 1 \
  -o $out/full_${tag}_tcf python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo full_rc=$?
