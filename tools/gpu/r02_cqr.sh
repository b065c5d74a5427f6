set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cholqr.py -x -q 2>&1 | tail -30
timeout 200 python tools/time_cholqr.py 2>&1 | tail -8
