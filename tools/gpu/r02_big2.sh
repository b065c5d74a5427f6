timeout 600 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -2
SKL_PARITY_REPORT=gpurun_out/cfg4.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "cfg4" 2>&1 | tail -2
cat gpurun_out/cfg4.jsonl | tail -1 | cut -c1-400
timeout 300 python tools/time_cholqr.py 8192x1024 2>&1 | tail -1
