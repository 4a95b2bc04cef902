#!/bin/bash
# A/B of tcf build variants: operand stages / C slots (s4c3 = default build)
out=gpurun_out; mkdir -p $out
for v in s4c3 s5c2 s4c3 s5c2; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 600 python tools/tcf_stats.py 131072 2>&1 | head -1 | sed "s/^/$v /"
done > $out/ab_stages.txt
cat $out/ab_stages.txt
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/s5c2/libmixtile_b200.so timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_factor.py -m gpu -q -x 2>&1 | tail -2
