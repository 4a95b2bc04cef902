#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for r in 1 2; do timeout 200 python tools/kbench.py --n 65536 --t 2 --lookahead 1 2>&1 | grep -E "cholesky|upd32 "; done
timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky|upd32 |upd64 "
echo "== exact lo"; timeout 300 python tools/acc_krige.py
echo "== rna lo"; MIXTILE_LIB=paper_2003_05324_b200/_build/variants/lorna/libmixtile_b200.so timeout 300 python tools/acc_krige.py
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/lorna/libmixtile_b200.so timeout 300 python tools/acc_tf32.py
