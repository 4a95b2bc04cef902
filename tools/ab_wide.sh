#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "wide or cosched or cta_pair" 2>&1 | tail -2
for o in "12=0" "12=1" "12=0" "12=1"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
for o in "12=1" "12=0"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
MT_OPTS=10=0,12=1 timeout 600 ncu --set full --clock-control none -k regex:tc2w_update_kernel -s 20 -c 1 -o gpurun_out/full_r01i_tc2w python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo done
