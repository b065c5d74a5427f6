timeout 120 python tools/prof_kernels.py srht 2 > /dev/null 2>&1; echo plain rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:srht_reg -s 1 -c 1 \
  -o gpurun_out/r02_srht_full python tools/prof_kernels.py srht 2 > gpurun_out/srht_ncu.log 2>&1; echo ncu rc=$?
