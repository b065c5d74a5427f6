timeout 300 python -m pytest tests/test_gpu_cholqr.py -q 2>&1 | tail -4
