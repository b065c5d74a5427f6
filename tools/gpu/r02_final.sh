# end-of-round evidence: every GPU test (full-size parity report), both bench
# arms, per-config timings, headline launch list
set -x
mkdir -p gpurun_out
SKL_PARITY_REPORT=gpurun_out/r02_parity_fullsize.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.out 2>&1; echo ref rc=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs.err; echo cfg rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-solve --no-e2e --no-parity > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
SKL_PROF_WARM_S=0.01 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_cqr_launches.csv python tools/prof_qr.py 2048 256 2 cholqr > /dev/null 2>&1; echo ncu2 rc=$?
SKL_PROF_WARM_S=0.01 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_cqr_big_launches.csv python tools/prof_qr.py 8192 1024 1 cholqr > /dev/null 2>&1; echo ncu3 rc=$?
timeout 300 python tools/time_cholqr.py 800x200 2048x256 2048x511 8192x511 2048x600 8192x1024 > gpurun_out/r02_time_cholqr.jsonl 2>&1; echo tc rc=$?
SKL_NO_PDL=1 timeout 300 python tools/prof_cqr_kernels.py 8192 1024 10 > gpurun_out/r02_cqr_kernels_8192.txt 2>&1
SKL_NO_PDL=1 timeout 300 python tools/prof_cqr_kernels.py 2048 256 20 1e8 > gpurun_out/r02_cqr_kernels_2048_k1e8.txt 2>&1
