#!/bin/bash
out=gpurun_out; mkdir -p $out
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_r02l.txt 2>&1; echo smoke_rc=$?
timeout 1500 python bench.py --steps 2 --warmup 3 > $out/bench_r02l.json 2> $out/bench_r02l.err; echo bench_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -c 5300 --csv --log-file $out/launches_r02l_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dp --no-e2e > $out/bench_under_ncu_r02l.log 2>&1
echo launches_rc=$?
