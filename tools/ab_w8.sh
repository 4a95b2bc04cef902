#!/bin/bash
for v in w8s2 w8s3c2; do MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "wide" 2>&1 | tail -1; done
for r in 1 2; do
  timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/base /'
  for v in w8s2 w8s3c2; do MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed "s/^/$v /"; done
done
timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/base /'
for v in w8s2 w8s3c2; do MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed "s/^/$v /"; done
