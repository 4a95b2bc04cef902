#!/bin/bash
# tests + bench + ncu of the hot kernels (current code)
tag=${1:-r01c}
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gpu_tests_$tag.log 2>&1; echo tests_rc=$?; tail -2 $out/gpu_tests_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo bench_rc=$?
for k in tc2_update_kernel dmma_tma_update_kernel gen_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 30 -c 2 \
    -o $out/full_${tag}_$k python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 \
    > $out/ncu_${tag}_$k.log 2>&1
done
echo done
