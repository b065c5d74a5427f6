timeout 600 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_fullsize.py tests/test_gpu_api_properties.py -q 2>&1 | tail -2
cat gpurun_out/par.jsonl 2>/dev/null | head -0
timeout 300 python tools/time_cholqr.py 800x200 2048x256 8192x1024 2>&1 | tail -3
