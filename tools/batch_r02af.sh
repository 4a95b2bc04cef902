#!/bin/bash
# re-tune super-column width (6) and band co-scheduling share (11) on the final kernel
out=gpurun_out; mkdir -p $out
timeout 1500 python tools/ab_opts.py 6 8,12,16 262144 8 1 > $out/ab_sw_final2.jsonl 2>&1; cut -c1-120 $out/ab_sw_final2.jsonl
timeout 1500 python tools/ab_opts.py 11 80,90,100 262144 8 1 > $out/ab_pct_final2.jsonl 2>&1; cut -c1-120 $out/ab_pct_final2.jsonl
