set -x
mkdir -p gpurun_out
python tools/bench_configs.py --reps 10 > gpurun_out/r02_bench_configs.jsonl 2> gpurun_out/r02_bench_configs.err; echo rc=$?
cat gpurun_out/r02_bench_configs.jsonl
python tools/prof_qr.py 2048 257 1 > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_qr_2048x257_launches.csv python tools/prof_qr.py 2048 257 0 > /dev/null 2>&1; echo ncu rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_qr_8192x1024_launches.csv python tools/prof_qr.py 8192 1024 0 > /dev/null 2>&1; echo ncu rc=$?
