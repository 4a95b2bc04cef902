#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in s4c3 bk32; do
  MIXTILE_LIB=paper_2003_05324_b200/_build/variants/$v/libmixtile_b200.so timeout 900 python tools/ab_opts.py 16 0 65536,131072,262144 8 1 2>&1 | sed "s/^/$v /"
done > $out/ab_bk32b.txt
cat $out/ab_bk32b.txt
