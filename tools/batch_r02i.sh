#!/bin/bash
# A/B of the tcf slab width (default BK=16/4 stages vs BK=32/2 stages, SWIZZLE_128B)
out=gpurun_out; mkdir -p $out
bash tools/build_variant.sh bk16 > /dev/null 2>&1 || true
for v in s4c3 bk32 s4c3 bk32; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 600 python tools/tcf_stats.py 131072 2>&1 | head -1 | sed "s/^/$v /"
done > $out/ab_bk32.txt
cat $out/ab_bk32.txt
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/bk32/libmixtile_b200.so timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -2
