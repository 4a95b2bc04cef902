#!/bin/bash
tag=${1:-r01h}
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/gpu_tests_$tag.log 2>&1; echo tests_rc=$?; tail -2 $out/gpu_tests_$tag.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo bench_rc=$?
MT_OPTS=10=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2_update_kernel -s 30 -c 2 \
  -o $out/full_${tag}_tc2 python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 2 \
  -o $out/full_${tag}_gen python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmma_tma_update_kernel -s 30 -c 1 \
  -o $out/full_${tag}_dmma python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo done
