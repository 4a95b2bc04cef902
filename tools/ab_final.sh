#!/bin/bash
for o in "11=90" "11=70" "11=110" "11=90"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
