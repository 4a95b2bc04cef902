#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gpu_tests_final2.log 2>&1; echo tests_rc=$?; tail -2 $out/gpu_tests_final2.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > $out/bench_final2.json 2> $out/bench_final2.err; echo bench_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tc2w_update_kernel -c 600 --csv --log-file $out/traffic_final_tc2w.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
MT_OPTS=10=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2w_update_kernel -s 20 -c 1 \
  -o $out/full_final_tc2w python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo done
