#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 2000 python tools/ab_lookahead.py 262144 > $out/ab_lookahead_262144.jsonl 2>&1; cut -c1-140 $out/ab_lookahead_262144.jsonl
