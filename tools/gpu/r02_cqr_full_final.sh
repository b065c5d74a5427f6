SKL_PROF_WARM_S=0.01 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cqr_gram" -s 2 -c 1 \
  -o gpurun_out/r02_cqr8192_gram_full python tools/prof_qr.py 8192 1024 1 cholqr > gpurun_out/cqr8192_g.log 2>&1; echo rc=$?
SKL_PROF_WARM_S=0.01 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"trsm_df_batch" -s 1 -c 1 \
  -o gpurun_out/r02_cqr8192_rinv_full python tools/prof_qr.py 8192 1024 1 cholqr > gpurun_out/cqr8192_r.log 2>&1; echo rc=$?
