# QR iteration: build, QR/solve parity tests, timings, probe + timeline builds
set -x
python -c "from paper_2409_14309_b200 import _build; _build.build()"
python -m pytest tests/test_gpu_parity.py -q -x -k "qr or solve or lsqr or sap or saa" 2>&1 | tail -3
for i in 1 2; do python tools/prof_qr.py 2048 257 3; python tools/prof_qr.py 8192 1024 3; python tools/prof_qr.py 800 201 3; done
SKL_NVCC_DEFINES="-DSKL_QR_PROBE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 2048 257 1 2>&1 | tail -2
python tools/prof_qr.py 8192 1024 1 2>&1 | tail -2
SKL_NVCC_DEFINES="-DSKL_QR_TIMELINE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 2048 257 2 2>&1 | tail -2
python tools/prof_qr.py 8192 1024 2 2>&1 | tail -2
