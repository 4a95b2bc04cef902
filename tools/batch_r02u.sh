#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python tools/tcf_stats.py 131072 2>&1 | head -1
timeout 1800 python tools/ab_opts.py 4 64,32,128 262144 8 1 > $out/ab_pcol.jsonl 2>&1; cut -c1-120 $out/ab_pcol.jsonl
