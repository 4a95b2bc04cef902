#!/bin/bash
out=gpurun_out; mkdir -p $out
./tools/sc_check
for v in 0 8 0 8; do timeout 900 python tools/ab_opts.py 6 $v 262144 8 1 2>&1 | grep '"round": 0'; done > $out/ab_sc_262144.txt
timeout 900 python tools/ab_opts.py 6 0,4,8,16 131072 8 1 > $out/ab_sc_131072.txt 2>&1
cut -c1-130 $out/ab_sc_262144.txt; cut -c1-130 $out/ab_sc_131072.txt
