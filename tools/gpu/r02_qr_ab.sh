set -x
for defs in "-DSKL_QR_PROBE" "-DSKL_QR_PROBE -DQR_SHFL_BCAST"; do
  SKL_NVCC_DEFINES="$defs" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
  python tools/prof_qr.py 8192 1024 1 2>&1 | tail -2
  python tools/prof_qr.py 2048 257 1 2>&1 | tail -2
done
for defs in "" "-DQR_SHFL_BCAST"; do
  SKL_NVCC_DEFINES="$defs" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
  for i in 1 2 3; do python tools/prof_qr.py 8192 1024 3; python tools/prof_qr.py 2048 257 3; done
done
