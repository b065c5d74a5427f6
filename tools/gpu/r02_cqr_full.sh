timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cqr_(gram|chol|trsm|solve_b)" -c 4 \
  -o gpurun_out/r02_cqr_full python tools/time_cholqr.py 2048x256 > gpurun_out/cqr_full.log 2>&1; echo rc=$?
