set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probgen.py tests/test_gpu_fullsize.py -q -x -k "lsqr or sap or dispatcher or solve" 2>&1 | tail -3
python tools/check_determinism.py 5 2>&1 | tail -1
for v in 1 "" 1 ""; do SKL_LSQR_FUSED_REG=$v python tools/bench_sap.py 2 2>&1 | tail -1 | cut -c1-200; done
ncu --set full --clock-control none -k regex:lsqr_fused_async -s 3 -c 1 -o gpurun_out/r02_lsqr_async_full python tools/bench_sap.py 2 > /dev/null 2>&1; echo ncu rc=$?
