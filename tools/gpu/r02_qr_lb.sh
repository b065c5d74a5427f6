set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "qr or solve or saa or cfg4 or cfg3" 2>&1 | tail -3
for i in 1 2; do python tools/prof_qr.py 8192 1024 10; python tools/prof_qr.py 4200 512 10; python tools/prof_qr.py 10000 1024 5; python tools/prof_qr.py 2048 257 20; done
SKL_NVCC_DEFINES="-DSKL_QR_PROBE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 8192 1024 1 2>&1 | tail -2
python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
