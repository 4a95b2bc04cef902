#!/bin/bash
# 16 epilogue warps (4 per TMEM lane quadrant, 64 columns each, 8-column C chunks) vs 8
out=gpurun_out; mkdir -p $out
V=paper_2003_05324_b200/_build/variants/epi16/libmixtile_b200.so
MIXTILE_LIB=$V timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_factor.py -m gpu -q -x > $out/gputest_r02ab.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02ab.txt
MIXTILE_LIB=$V timeout 900 python tools/tcf_stats.py 131072 2>&1 | tail -2
for r in 0 1; do
  timeout 1200 python tools/ab_opts.py 17 1 131072,262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"epi8\", /" >> $out/ab_epi16.jsonl
  MIXTILE_LIB=$V timeout 1200 python tools/ab_opts.py 17 1 131072,262144 8 1 2>&1 | sed 's/^{/{"lib": "epi16", /' >> $out/ab_epi16.jsonl
done
cut -c1-190 $out/ab_epi16.jsonl
