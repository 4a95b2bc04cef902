#!/bin/bash
out=gpurun_out; mkdir -p $out
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/cw8s4/libmixtile_b200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_factor.py tests/test_gpu_predict.py -m gpu -q -x 2>&1 | tail -2
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/cw8s4/libmixtile_b200.so timeout 600 python tools/tcf_stats.py 131072 2>&1 | head -1
for v in dflt cw8s4 dflt cw8s4; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 900 python tools/ab_opts.py 16 0 131072,262144 8 1 2>&1 | grep '"round": 0' | sed "s/^/$v /"
done > $out/ab_cw8.txt
cut -c1-130 $out/ab_cw8.txt
