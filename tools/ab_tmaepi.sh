#!/bin/bash
V=paper_2003_05324_b200/_build/variants/noTmaEpi/libmixtile_b200.so
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_factor.py tests/test_gpu_mle.py -q -x 2>&1 | tail -2
for r in 1 2; do
  timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky"
  MIXTILE_LIB=$V timeout 200 python tools/kbench.py --n 131072 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/old /'
done
timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky|upd"
MIXTILE_LIB=$V timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead 1 2>&1 | grep -E "cholesky" | sed 's/^/old /'
timeout 300 ncu --set full --clock-control none -k regex:tc2_update_kernel -s 30 -c 1 -o gpurun_out/full_r01g_tc2 python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
echo done
