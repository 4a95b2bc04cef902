#!/bin/bash
# TMEM drain with x32 loads (one wait per 32 columns) vs x16; full ncu capture of a bulk launch
out=gpurun_out; mkdir -p $out
V=paper_2003_05324_b200/_build/variants/ldx32/libmixtile_b200.so
MIXTILE_LIB=$V timeout 900 python -m pytest tests/test_gpu_tc.py -m gpu -q -x -k "bitwise" > $out/gputest_r02ad.txt 2>&1; echo t_rc=$?; tail -1 $out/gputest_r02ad.txt
for r in 0 1; do
  timeout 1200 python tools/ab_opts.py 17 1 131072,262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"ldx16\", /" >> $out/ab_ldx32.jsonl
  MIXTILE_LIB=$V timeout 1200 python tools/ab_opts.py 17 1 131072,262144 8 1 2>&1 | sed "s/^{/{\"lib\": \"ldx32\", /" >> $out/ab_ldx32.jsonl
done
cut -c1-190 $out/ab_ldx32.jsonl
MT_OPTS=10=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcf_update_kernel -s 81 -c 1 \
  -o $out/full_r02ad_tcf_bulk python tools/prof_eval.py --n 131072 --t 8 --warm 0 --reps 1 > /dev/null 2>&1; echo full_rc=$?
