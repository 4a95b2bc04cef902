#!/bin/bash
# round 2: warp-level diagonal-block factor + inverse in every POTRF variant
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -x -q > $out/gputest_r02z.txt 2>&1; echo t_rc=$?; tail -3 $out/gputest_r02z.txt
for o in 0 1 2; do MT_OPTS=14=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 200 --csv \
  --log-file $out/potrf_z_opt$o.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; done
for o in 0 1 2; do python tools/launch_summary.py $out/potrf_z_opt$o.csv; done
timeout 1500 python tools/ab_opts.py 14 0,2 131072,262144 8 1 > $out/ab_potrf_z.jsonl 2>&1; cut -c1-150 $out/ab_potrf_z.jsonl
