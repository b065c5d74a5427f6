timeout 600 python -m pytest tests/test_gpu_api_properties.py tests/test_gpu_cholqr.py tests/test_gpu_multidevice.py -q 2>&1 | tail -2
timeout 300 python tools/time_solve.py 2 2>&1 | tail -2
timeout 300 python tools/prof_solve_host.py 2>&1 | sed -n 1,16p
