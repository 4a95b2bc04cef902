timeout 300 python -m pytest tests/test_gpu_predict.py -q 2>&1 | tail -3
DIAG=0,1,2,3,4,0 timeout 300 python tools/diag_tc32.py 65536
DIAG=0 EXTRA="6=16;6=0,7=1;7=0" timeout 300 python tools/diag_tc32.py 65536
DIAG=0,1,4 timeout 300 python tools/diag_tc32.py 131072
