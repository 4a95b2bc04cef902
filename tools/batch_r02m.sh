#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in dflt s3w16 dflt s3w16; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 900 python tools/ab_opts.py 16 0 65536,131072 8 1 2>&1 | sed "s/^/$v /"
done > $out/ab_s3w16.txt
cat $out/ab_s3w16.txt | cut -c1-150
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/s3w16/libmixtile_b200.so timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_factor.py tests/test_gpu_predict.py -m gpu -q -x 2>&1 | tail -2
