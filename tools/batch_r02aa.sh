#!/bin/bash
# option 17: C update by TMA reduce-add -- bitwise test, A/B timing, issuer stats
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_tc.py -m gpu -q -k "reduce_add or four_cta" > $out/gputest_r02aa.txt 2>&1; echo t_rc=$?; tail -3 $out/gputest_r02aa.txt
timeout 900 python tools/tcf_stats.py 131072 2>&1 | tail -2
timeout 2400 python tools/ab_opts.py 17 0,1 131072,262144 8 2 > $out/ab_tcf_reduce.jsonl 2>&1; cut -c1-200 $out/ab_tcf_reduce.jsonl
