#!/bin/bash
# L2 eviction-priority hints on the FP32 update (B evict_last, C reduce evict_first)
out=gpurun_out; mkdir -p $out
V=paper_2003_05324_b200/_build/variants/l2hint/libmixtile_b200.so
MIXTILE_LIB=$V timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q -x -k "reduce_add" > $out/gputest_r02am.txt 2>&1; echo t_rc=$?; tail -1 $out/gputest_r02am.txt
for r in 0 1; do
  timeout 900 python tools/ab_opts.py 17 1 262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"nohint\", /" >> $out/ab_l2hint.jsonl
  MIXTILE_LIB=$V timeout 900 python tools/ab_opts.py 17 1 262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"l2hint\", /" >> $out/ab_l2hint.jsonl
done
cut -c1-150 $out/ab_l2hint.jsonl
