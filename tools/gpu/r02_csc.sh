set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multidevice.py -q -x -k "csr or sparse or cfg4 or lsqr" 2>&1 | tail -3
for v in 1 ""; do SKL_CSR_BUCKET_WALK=$v python tools/bench_configs.py --configs 4 2>&1 | tail -1; done
