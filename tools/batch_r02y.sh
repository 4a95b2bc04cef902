#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_factor.py -m gpu -q -k "potrf" > $out/gputest_r02y.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02y.txt
for o in 0 2; do MT_OPTS=14=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 200 --csv \
  --log-file $out/potrf_opt$o.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; done
python tools/launch_summary.py $out/potrf_opt0.csv; python tools/launch_summary.py $out/potrf_opt2.csv
timeout 1500 python tools/ab_opts.py 14 0,2 131072,262144 8 1 > $out/ab_potrf_mk.jsonl 2>&1; cut -c1-120 $out/ab_potrf_mk.jsonl
