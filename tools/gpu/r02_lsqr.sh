set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_properties.py tests/test_gpu_probgen.py -x -q -k "sap or lsqr or triangular or precond or direct or solve" 2>&1 | tail -3
SKL_LSQR_HOST_LOOP=1 python -m pytest tests/test_gpu_parity.py -x -q -k "sap or lsqr" 2>&1 | tail -2
for v in "" 1; do SKL_LSQR_HOST_LOOP=$v python tools/bench_sap.py 2 | cut -c1-300; done
SKL_LSQR_HOST_LOOP=1 SKL_LSQR_DTRTRS=1 python tools/bench_sap.py 2 | cut -c1-300
