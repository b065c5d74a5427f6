set -x
python -c "from paper_2409_14309_b200 import _build; _build.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "qr or solve or lsqr or sap or saa" 2>&1 | tail -3
for v in 1 "" 1 ""; do
  SKL_NO_PDL=$v python tools/prof_qr.py 2048 257 30
  SKL_NO_PDL=$v python tools/prof_qr.py 800 201 30
  SKL_NO_PDL=$v python tools/prof_qr.py 8192 1024 10
  SKL_NO_PDL=$v python tools/prof_qr.py 2048 513 20
done
