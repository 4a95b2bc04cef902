#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1200 python tools/ab_opts.py 15 0,1 131072,262144 8 1 > $out/ab_c4_bk32.jsonl 2>&1; cat $out/ab_c4_bk32.jsonl | cut -c1-120
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest_r02k.txt 2>&1; echo tests_rc=$?; tail -3 $out/gputest_r02k.txt
