timeout 600 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -3
timeout 300 python tools/time_cholqr.py 800x200 2048x256 2048x600 8192x1024 2>&1 | tail -4
SKL_CQR_SINGLE=1 timeout 300 python tools/time_cholqr.py 800x200 2048x256 2048x600 8192x1024 2>&1 | tail -4
SKL_NO_PDL=1 timeout 300 python tools/prof_cqr_kernels.py 8192 1024 2>&1 | tail -18
