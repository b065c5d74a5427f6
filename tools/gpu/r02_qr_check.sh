set -x
python -c "from paper_2409_14309_b200 import _build; _build.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "qr or solve or lsqr or sap or saa or cfg" 2>&1 | tail -4
python tools/prof_qr.py 2048 257 30; python tools/prof_qr.py 8192 1024 10
