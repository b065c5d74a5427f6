timeout 600 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -1
for sb in 0 9 7; do SKL_CQR_SB=$sb timeout 300 python tools/time_cholqr.py 2048x600 8192x1024 2>&1 | grep '"d"'; done
