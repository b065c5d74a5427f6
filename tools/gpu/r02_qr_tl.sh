# QR critical-path timeline (instrumented build): full, no bulk, no next-panel updates
set -x
SKL_NVCC_DEFINES="-DSKL_QR_TIMELINE" python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
for skip in 0 1; do
  SKL_QR_SKIP=$skip python tools/prof_qr.py 8192 1024 2 2>&1 | tail -9
  SKL_QR_SKIP=$skip python tools/prof_qr.py 2048 257 2 2>&1 | tail -9
done
python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
