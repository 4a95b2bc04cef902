#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 2400 python tools/ab_opts.py 11 90,75,105 262144 8 1 > $out/ab_pct2.jsonl 2>&1; cut -c1-120 $out/ab_pct2.jsonl
timeout 1200 python tools/ab_opts.py 6 8,12,16 262144 8 1 > $out/ab_sw2.jsonl 2>&1; cut -c1-120 $out/ab_sw2.jsonl
