#!/bin/bash
# round-2 batch: configs[1]-scale parity field, configs[2] band search, configs[4] MLE, GPU tests
out=gpurun_out; mkdir -p $out
timeout 600 python tools/make_field65536.py $out/field65536_gpu.npz > $out/field65536_gpu.log 2>&1; echo field_rc=$?
timeout 900 python tools/config3_band_gpu.py 131072 > $out/config3_band_gpu.jsonl 2> $out/config3_band_gpu.err; echo c3_rc=$?
BANDS=2,8,13 SAVE=$out/mle_config5_data.npz timeout 2400 python tools/mle_config5.py > $out/mle_config5_r02.json 2> $out/mle_config5_r02.err; echo mle_rc=$?
timeout 900 python -m pytest tests -m gpu -q -rs > $out/gputest_r02b.txt 2>&1; echo tests_rc=$?; tail -5 $out/gputest_r02b.txt
