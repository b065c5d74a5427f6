set -x
for i in 1 2 3; do python tools/prof_qr.py 8192 1024 3; python tools/prof_qr.py 2048 257 3; done
for rows in 256 512; do
  for i in 1 2; do SKL_QR_PANEL_ROWS=$rows python tools/prof_qr.py 2048 257 3; SKL_QR_PANEL_ROWS=$rows python tools/prof_qr.py 2048 513 3; SKL_QR_PANEL_ROWS=$rows python tools/prof_qr.py 800 201 3; done
done
python tools/prof_qr.py 2048 513 3; python tools/prof_qr.py 800 201 3
SKL_NVCC_DEFINES="-DSKL_QR_PROBE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 8192 1024 1 2>&1 | tail -2
SKL_QR_PANEL_ROWS=512 python tools/prof_qr.py 2048 257 1 2>&1 | tail -2
