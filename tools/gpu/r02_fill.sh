SKL_PROF_WARM_S=0.01 timeout 600 ncu --set full --import-source on --clock-control none -k regex:owned_fill -s 1 -c 1 \
  -o gpurun_out/r02_fill python tools/prof_build.py 2 > /dev/null 2>&1; echo ncu rc=$?
