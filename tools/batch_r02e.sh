#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_tc.py -m gpu -q -k "tcf_four or tf32x3_factor or coscheduled" > $out/gputest_r02e.txt 2>&1; echo tests_rc=$?; tail -3 $out/gputest_r02e.txt
timeout 900 python tools/ab_opts.py 15 0,1 65536,131072 8 2 > $out/ab_cluster4.jsonl 2>&1; echo ab_rc=$?; cat $out/ab_cluster4.jsonl
