#!/bin/bash
# A/B timing of kernel variants (dev tool): serialized + lookahead Cholesky
set -x
for la in 0 1; do
  python tools/kbench.py --n 65536 --t 2 --lookahead $la --legacy-dmma 1 --tc-trsm 0
  python tools/kbench.py --n 65536 --t 2 --lookahead $la --legacy-dmma 0 --tc-trsm 0
  python tools/kbench.py --n 65536 --t 2 --lookahead $la --legacy-dmma 0 --tc-trsm 1
done
python tools/kbench.py --n 32768 --dp --legacy-dmma 1
python tools/kbench.py --n 32768 --dp --legacy-dmma 0
python tools/kbench.py --n 65536 --t 8 --lookahead 1 --legacy-dmma 0 --tc-trsm 1
