# e2e host-stream block size sweep, then the QR probe (instrumented build)
set -x
mkdir -p gpurun_out
for mb in 32 64 128 256; do
  SKL_HOST_BLOCK_MB=$mb python bench.py --steps 5 --warmup 3 --no-cpu --no-solve --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('blockMB', $mb, d['e2e'])"
done
python tools/prof_qr.py 8192 1024 3
python tools/prof_qr.py 2048 257 3
SKL_NVCC_DEFINES=-DSKL_QR_PROBE python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)"
python tools/prof_qr.py 8192 1024 1 2>&1 | tail -3
python tools/prof_qr.py 2048 257 1 2>&1 | tail -3
