#!/bin/bash
# multi-rank bench logic on one GPU (ranks share cuda:0 over gloo; NCCL refuses that)
out=gpurun_out; mkdir -p $out
MT_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --n 16384 --nb 512 --t 8 --steps 1 --warmup 3 --no-cpu --dp-n 8192 > $out/bench_gloo2.json 2> $out/bench_gloo2.err; echo rc2=$?
tail -c 1500 $out/bench_gloo2.json; tail -5 $out/bench_gloo2.err
MT_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 4 --grid 2x2 --n 16384 --nb 512 --t 8 --steps 1 --warmup 3 --no-cpu --dp-n 8192 > $out/bench_gloo4.json 2> $out/bench_gloo4.err; echo rc4=$?
tail -c 1500 $out/bench_gloo4.json; tail -5 $out/bench_gloo4.err
