#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for o in "13=0" "13=1" "13=0" "13=1"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
for o in "13=1" "13=0"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
