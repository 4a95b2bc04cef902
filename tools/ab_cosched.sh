#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "cosched or cta_pair" 2>&1 | tail -2
for o in "10=0" "10=1" "10=0" "10=1"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 65536 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
for o in "10=1" "10=0"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky|upd"
done
