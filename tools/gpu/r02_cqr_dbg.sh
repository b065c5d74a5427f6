timeout 300 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | grep -E "^(FAILED|ERROR)|Error|test_cholqr|\[" | head -20
