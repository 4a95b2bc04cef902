#!/bin/bash
# reduce-add epilogue without the C prefetch into L2: time and DRAM traffic
out=gpurun_out; mkdir -p $out
V=paper_2003_05324_b200/_build/variants/nopf/libmixtile_b200.so
MIXTILE_LIB=$V timeout 900 python -m pytest tests/test_gpu_tc.py -m gpu -q -x -k "reduce_add" > $out/gputest_r02aj.txt 2>&1; echo t_rc=$?; tail -1 $out/gputest_r02aj.txt
for r in 0 1; do
  timeout 1200 python tools/ab_opts.py 17 1 262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"prefetch\", /" >> $out/ab_nopf.jsonl
  MIXTILE_LIB=$V timeout 1200 python tools/ab_opts.py 17 1 262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"no_prefetch\", /" >> $out/ab_nopf.jsonl
done
cut -c1-150 $out/ab_nopf.jsonl
MIXTILE_LIB=$V timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:tcf_update_kernel -c 1100 --csv --log-file $out/traffic_r02aj_nopf.csv \
  python tools/prof_eval.py --n 262144 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; echo traffic_rc=$?
