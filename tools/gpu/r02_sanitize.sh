# compute-sanitizer over small-size tests of every kernel family (memcheck;
# racecheck/synccheck on the shared-memory kernels)
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 --target-processes all \
  python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py \
  -k "ragged or both_plans or few_long or cfg1 or misaligned or economy_qr or srht or gaussian or fwht or csr" \
  > gpurun_out/r02_memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/r02_memcheck.log
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest -x -q -p no:cacheprovider tests/test_gpu_slots.py -k "reduce_peers or emulated" \
  > gpurun_out/r02_memcheck_slots.log 2>&1; echo memcheck2 rc=$?
tail -3 gpurun_out/r02_memcheck_slots.log
timeout 900 $CS --tool racecheck --error-exitcode 9 \
  python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "cfg1_bitwise or economy_qr_matches or srht_cfg or few_long_columns_bitwise" \
  > gpurun_out/r02_racecheck.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/r02_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 \
  python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "cfg1_bitwise or economy_qr_matches or few_long_columns_bitwise" \
  > gpurun_out/r02_synccheck.log 2>&1; echo synccheck rc=$?
tail -3 gpurun_out/r02_synccheck.log
