#!/bin/bash
V=paper_2003_05324_b200/_build/variants/splitacc/libmixtile_b200.so
echo "== default"; timeout 300 python tools/acc_krige.py
echo "== splitacc"; MIXTILE_LIB=$V timeout 300 python tools/acc_krige.py
MIXTILE_LIB=$V timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_mle.py tests/test_gpu_predict.py -q 2>&1 | tail -3
timeout 300 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
MIXTILE_LIB=$V timeout 300 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/split /'
MIXTILE_LIB=$V timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/split /'
MIXTILE_LIB=$V T=2 timeout 600 python tools/mle_noise.py
