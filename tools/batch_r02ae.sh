#!/bin/bash
# retest option 15 (4-CTA clusters, B multicast: 25% less L2->SM operand traffic) on the final layout; DMMA capture
out=gpurun_out; mkdir -p $out
timeout 2400 python tools/ab_opts.py 15 0,1 131072,262144 8 1 > $out/ab_cluster4_final.jsonl 2>&1; cut -c1-170 $out/ab_cluster4_final.jsonl
MT_OPTS=10=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_tma_update_kernel -s 40 -c 1 \
  -o $out/full_r02ae_dmma python tools/prof_eval.py --n 131072 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; echo full_rc=$?
