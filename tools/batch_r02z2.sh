#!/bin/bash
# diagonal block: rolled (default) vs fully unrolled pivot loop
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_factor.py -m gpu -q -k "potrf" > $out/gputest_r02z2.txt 2>&1; echo t_rc=$?; tail -1 $out/gputest_r02z2.txt
V=paper_2003_05324_b200/_build/variants/potrf_unrolled/libmixtile_b200.so
for o in 0 1 2; do
  MT_OPTS=14=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 200 --csv \
    --log-file $out/potrf_z2_opt$o.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
  MIXTILE_LIB=$V MT_OPTS=14=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -c 200 --csv \
    --log-file $out/potrf_z2u_opt$o.csv python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
done
for o in 0 1 2; do echo "== rolled opt $o"; python tools/launch_summary.py $out/potrf_z2_opt$o.csv; echo "== unrolled opt $o"; python tools/launch_summary.py $out/potrf_z2u_opt$o.csv; done
MT_OPTS=14=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:potrf_mk_diag -s 20 -c 1 -o $out/potrf_mk_diag_full python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 > /dev/null 2>&1
ls -la $out/potrf_mk_diag_full*
