timeout 300 python -m pytest tests/test_gpu_cholqr.py -q 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cqr_(gram|trsm)" -c 2 \
  -o gpurun_out/r02_cqr_gram python tools/time_cholqr.py 2048x256 > gpurun_out/cqr_full.log 2>&1; echo rc=$?
