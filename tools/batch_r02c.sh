#!/bin/bash
# round-2 batch c: full GPU tests (P x Q distributed, cluster POTRF, integration), option A/Bs,
# ncu capture of the bulk tcf update and POTRF per-tile times
out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs > $out/gputest_r02c.txt 2>&1; echo tests_rc=$?; tail -5 $out/gputest_r02c.txt
timeout 900 python tools/ab_opts.py 6 0,4,8 65536,131072 8 2 > $out/ab_supercols.jsonl 2>&1; echo ab6_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 60 --csv \
  --log-file $out/potrf_cluster.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
MT_OPTS=14=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 60 --csv \
  --log-file $out/potrf_single.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo potrf_rc=$?
MT_OPTS=10=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcf_update_kernel -s 21 -c 1 \
  -o $out/full_r02c_tcf python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo full_rc=$?
