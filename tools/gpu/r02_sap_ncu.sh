mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_sap_launches.csv python tools/bench_sap.py 2 > /dev/null 2>&1; echo rc=$?
