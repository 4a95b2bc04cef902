#!/bin/bash
# final-tree validation: smoke, full GPU suite, reference arm (short)
out=gpurun_out; mkdir -p $out
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke_r02ag.txt 2>&1; echo smoke_rc=$?; tail -2 $out/smoke_r02ag.txt
timeout 2400 python -m pytest tests -m gpu -q > $out/gputest_r02ag.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02ag.txt
timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > $out/bench_ref_r02ag.json 2> $out/bench_ref_r02ag.err; echo ref_rc=$?; tail -c 400 $out/bench_ref_r02ag.json
