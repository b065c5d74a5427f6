timeout 300 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -3
timeout 200 python tools/time_cholqr.py 800x200 2048x256 2048x511 8192x511 2>&1 | tail -4
export SKL_NVCC_DEFINES=-DSKL_CQR_PROBE
python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)" 2>&1 | tail -2
timeout 120 python tools/probe_cholqr.py 2048x256 2>&1 | head -4 | cut -c1-300
