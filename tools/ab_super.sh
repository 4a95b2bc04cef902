#!/bin/bash
# A/B of the FP32 update output order (option 6) and the C-block L2 prefetch (option 7)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_ab.log 2>&1; echo tests_rc=$?; grep -E "passed|failed|Error|assert" gpurun_out/gpu_tests_ab.log | head -20
for o in "6=0,7=0" "6=0,7=1" "6=16,7=1" "6=8,7=1"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 65536 --t 2 --lookahead 1 2>&1 | head -7
done
for o in "6=0,7=1" "6=16,7=1"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | head -7
done
