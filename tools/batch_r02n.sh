#!/bin/bash
# interleaved same-box A/B at the bench size: default (32-col slabs) vs 16-col slabs
out=gpurun_out; mkdir -p $out
for v in dflt bk16 s3w16 dflt bk16 s3w16; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 900 python tools/ab_opts.py 16 0 262144 8 1 2>&1 | grep '"round": 0' | sed "s/^/$v /"
done > $out/ab_bk_262144.txt
cat $out/ab_bk_262144.txt | cut -c1-140
