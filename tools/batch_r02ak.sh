#!/bin/bash
# final tree (no C prefetch): full GPU suite, smoke, default bench line
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q > $out/gputest_r02ak.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02ak.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke_r02ak.txt 2>&1; echo smoke_rc=$?; tail -1 $out/smoke_r02ak.txt
timeout 1500 python bench.py > $out/bench_r02ak.json 2> $out/bench_r02ak.err; echo bench_rc=$?; tail -c 300 $out/bench_r02ak.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -c 5300 --csv --log-file $out/launches_r02ak_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-dp --no-e2e > $out/bench_under_ncu_r02ak.log 2>&1; echo launches_rc=$?
