#!/bin/bash
# super-column width after dropping the C prefetch
out=gpurun_out; mkdir -p $out
timeout 1500 python tools/ab_opts.py 6 12,16,8 262144 8 1 > $out/ab_sw_nopf.jsonl 2>&1; cut -c1-120 $out/ab_sw_nopf.jsonl
