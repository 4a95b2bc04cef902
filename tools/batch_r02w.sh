#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest_r02w.txt 2>&1; echo tests_rc=$?; tail -2 $out/gputest_r02w.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke_r02w.txt 2>&1; echo smoke_rc=$?; tail -2 $out/smoke_r02w.txt
timeout 1500 python bench.py > $out/bench_r02w.json 2> $out/bench_r02w.err; echo bench_rc=$?
timeout 1500 python bench.py --impl reference --steps 1 --warmup 1 > $out/bench_ref_r02w.json 2> $out/bench_ref_r02w.err; echo ref_rc=$?; tail -c 600 $out/bench_ref_r02w.json
