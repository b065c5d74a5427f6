set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probgen.py -q -x -k "lsqr or sap or dispatcher or solve" 2>&1 | tail -3
python tools/check_determinism.py 10 2>&1 | tail -3
for v in 1 "" 1 ""; do SKL_NO_PDL=$v python tools/bench_sap.py 2 2>&1 | tail -1; done
