timeout 600 python -m pytest tests/test_gpu_cholqr.py -q 2>&1 | tail -2
timeout 300 python tools/time_cholqr.py 800x200 2048x256 8192x1024 2>&1 | tail -3
SKL_CQR_TRSM_LL=1 timeout 300 python tools/time_cholqr.py 800x200 2048x256 8192x1024 2>&1 | tail -3
