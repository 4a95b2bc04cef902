timeout 600 python tools/acc_tf32.py
MIXTILE_LIB=paper_2003_05324_b200/_build/variants/lotrunc/libmixtile_b200.so timeout 600 python tools/acc_tf32.py
timeout 300 python -m pytest tests/test_gpu_predict.py -q 2>&1 | grep -E "^E  |passed|failed" | head -20
