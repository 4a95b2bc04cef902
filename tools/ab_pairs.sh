#!/bin/bash
# correctness of the CTA-pair kernel, then A/B timing vs the single-CTA kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
DIAG=0 EXTRA="9=0;9=1;9=0;9=1" timeout 300 python tools/diag_tc32.py 65536
for o in "9=0" "9=1" "9=0" "9=1"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 65536 --t 2 --lookahead 1 2>&1 | head -7
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for o in "9=1" "9=0"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | head -7
done
