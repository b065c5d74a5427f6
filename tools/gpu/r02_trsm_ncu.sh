SKL_PROF_WARM_S=0.01 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cqr_trsm_df" -s 2 -c 1 \
  -o gpurun_out/r02_trsm_df_full python tools/prof_qr.py 8192 1024 1 cholqr > gpurun_out/trsm_f.log 2>&1; echo rc=$?
tail -2 gpurun_out/trsm_f.log
