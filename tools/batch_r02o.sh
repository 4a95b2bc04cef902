#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest_r02o.txt 2>&1; echo tests_rc=$?; tail -2 $out/gputest_r02o.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_r02o.txt 2>&1; echo smoke_rc=$?; tail -2 $out/smoke_r02o.txt
timeout 1500 python tools/ab_opts.py 0 1,2 262144 8 1 > $out/ab_engine_262144.jsonl 2>&1; cut -c1-140 $out/ab_engine_262144.jsonl
timeout 1500 python bench.py --steps 2 --warmup 3 > $out/bench_r02o.json 2> $out/bench_r02o.err; echo bench_rc=$?
