#!/bin/bash
V=paper_2003_05324_b200/_build/variants/epi8/libmixtile_b200.so
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
MIXTILE_LIB=$V timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
for r in 1 2; do
for o in "6=0" "6=16"; do
  MT_OPTS=$o timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
  MIXTILE_LIB=$V MT_OPTS=$o timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/epi8 /'
done
done
timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
MIXTILE_LIB=$V timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/epi8 /'
