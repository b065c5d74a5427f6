timeout 300 python tools/time_solve.py 2 2>&1 | tail -3
SKL_PROF_WARM_S=0.01 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_cqr_launches.csv python tools/prof_qr.py 2048 256 2 cholqr > gpurun_out/cqr_l.log 2>&1; echo rc=$?
SKL_PROF_WARM_S=0.01 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cqr_(gram|chol|trsm)" -s 9 -c 3 \
  -o gpurun_out/r02_cholqr_full python tools/prof_qr.py 2048 256 2 cholqr > gpurun_out/cqr_f.log 2>&1; echo rc=$?
