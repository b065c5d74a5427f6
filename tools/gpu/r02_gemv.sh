timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_api_properties.py -q -k "gaussian or cfg3" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py 3 2>&1 | tail -1 | cut -c1-400
