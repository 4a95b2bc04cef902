#!/bin/bash
for o in "10=1,11=60" "10=1,11=90" "10=1,11=120" "10=1,11=160" "10=0"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
for o in "10=1,11=130" "10=1,11=90"; do
  MT_OPTS=$o timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
done
