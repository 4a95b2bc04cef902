#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_factor.py -m gpu -q -x > $out/gputest_r02f.txt 2>&1; echo tests_rc=$?; tail -3 $out/gputest_r02f.txt
timeout 1500 python tools/ab_opts.py 11 90,105,120,140 131072,262144 8 1 > $out/ab_cosched_pct.jsonl 2>&1; echo ab_rc=$?; cat $out/ab_cosched_pct.jsonl
