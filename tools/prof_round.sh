#!/bin/bash
# One profiling pass (run under gpurun): serialized + pipelined kernel breakdown,
# ncu --set full of the hot kernels, and the launch list of a bench command.
#   bash tools/prof_round.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# serialized (lookahead 0) and pipelined breakdowns at the bench config
for la in 0 1; do
  timeout 300 python tools/kbench.py --n 262144 --t 8 --lookahead $la > $out/kbench_${tag}_la$la.txt 2>&1
done
# ncu --set full: bulk 3xTF32 update, DMMA band update, POTRF (3 launches each, mid-factorization)
for k in tc32_update_kernel dmma_update_kernel potrf_kernel tc32_trsm_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 3 \
    -o $out/full_${tag}_$k python tools/prof_eval.py --n 65536 --t 8 --warm 0 --reps 1 \
    > $out/ncu_${tag}_$k.log 2>&1
done
# launch list of the bench command (serialised cold-cache device times)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 7000 --csv --log-file $out/launches_${tag}_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dp --no-e2e > $out/bench_under_ncu.log 2>&1
echo done
