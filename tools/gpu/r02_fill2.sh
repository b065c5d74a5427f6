timeout 120 python tools/prof_build.py 6 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "build or plan or owned or hash" 2>&1 | tail -2
