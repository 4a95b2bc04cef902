#!/bin/bash
# ncu launch list (device time + DRAM bytes + grid) of the bench command's first evaluation
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -c 5300 --csv --log-file gpurun_out/launches_${1:-r01e}_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dp --no-e2e > gpurun_out/bench_under_ncu_${1:-r01e}.log 2>&1
echo rc=$?
