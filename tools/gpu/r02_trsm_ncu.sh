SKL_PROF_WARM_S=0.01 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cqr_trsm_rl" -s 2 -c 2 \
  -o gpurun_out/r02_trsm_full2 python tools/prof_qr.py 8192 1024 1 cholqr > gpurun_out/trsm_f.log 2>&1; echo rc=$?
tail -3 gpurun_out/trsm_f.log
