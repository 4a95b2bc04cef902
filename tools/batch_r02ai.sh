#!/bin/bash
# super-column width 12 default: full GPU suite + default bench line
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q > $out/gputest_r02ai.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02ai.txt
timeout 1500 python bench.py > $out/bench_r02ai.json 2> $out/bench_r02ai.err; echo bench_rc=$?; tail -c 300 $out/bench_r02ai.err
