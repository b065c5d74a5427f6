# round-2 validation: every GPU test (incl. full-size parity), both bench arms,
# the headline launch list, a QR launch list
set -x
mkdir -p gpurun_out
SKL_PARITY_REPORT=gpurun_out/r02_parity_fullsize.jsonl python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.out 2>&1; echo ref rc=$?
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-solve --no-e2e --no-parity > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
