#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_factor.py -m gpu -q -k "lookahead" > $out/gputest_r02h_la.txt 2>&1; echo la_rc=$?; tail -2 $out/gputest_r02h_la.txt
timeout 900 python tools/ab_lookahead.py 131072 > $out/ab_lookahead.jsonl 2>&1; cat $out/ab_lookahead.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest_r02h.txt 2>&1; echo tests_rc=$?; tail -3 $out/gputest_r02h.txt
