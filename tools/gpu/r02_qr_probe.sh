set -x
SKL_NVCC_DEFINES="-DSKL_QR_PROBE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 2048 257 1 2>&1 | tail -3
python tools/prof_qr.py 8192 1024 1 2>&1 | tail -3
