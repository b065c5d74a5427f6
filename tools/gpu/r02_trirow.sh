timeout 600 python -m pytest tests/test_gpu_cholqr.py -q 2>&1 | tail -2
timeout 300 python tools/time_cholqr.py 2048x600 8192x1024 2>&1 | tail -2
