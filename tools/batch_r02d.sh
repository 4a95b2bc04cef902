#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > $out/gputest_r02d.txt 2>&1; echo tests_rc=$?; tail -3 $out/gputest_r02d.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_r02d.txt 2>&1; echo smoke_rc=$?
timeout 1500 python bench.py > $out/bench_r02d.json 2> $out/bench_r02d.err; echo bench_rc=$?
