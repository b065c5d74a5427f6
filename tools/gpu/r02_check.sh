set -x
mkdir -p gpurun_out
SKL_SKIP_FULLSIZE=1 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
tail -3 gpurun_out/r02_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_bench_ref.out 2>&1; echo ref rc=$?
python tools/prof_countsketch.py 2 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:countsketch_owned -s 2 -c 1 \
    -o gpurun_out/r02_cs_owned_full python tools/prof_countsketch.py 2 4 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-solve --no-e2e --no-parity > gpurun_out/ncu_launch.log 2>&1; echo ncu2 rc=$?
