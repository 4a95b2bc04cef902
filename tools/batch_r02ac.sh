#!/bin/bash
# final tree: full GPU suite + measurement pass
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q > $out/gputest_r02ac.txt 2>&1; echo t_rc=$?; tail -2 $out/gputest_r02ac.txt
bash tools/prof_r02.sh r02ac
