set -x
mkdir -p gpurun_out
python tools/prof_qr.py 8192 1024 3
python tools/prof_qr.py 2048 257 3
python tools/prof_qr.py 2048 513 3
python tools/prof_qr.py 800 201 3
python tools/time_solve.py 2
SKL_SKIP_FULLSIZE=1 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
