#!/bin/bash
V=paper_2003_05324_b200/_build/variants/cs5/libmixtile_b200.so
MIXTILE_LIB=$V timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "wide" 2>&1 | tail -1
for r in 1 2; do
  timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
  MIXTILE_LIB=$V timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/cs5 /'
done
timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
MIXTILE_LIB=$V timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/cs5 /'
