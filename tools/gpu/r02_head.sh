# re-entry check of HEAD: GPU tests (no full-size), bench line, config timings
set -x
mkdir -p gpurun_out
SKL_SKIP_FULLSIZE=1 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
tail -3 gpurun_out/r02_bench.err
timeout 900 python tools/bench_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs.err; echo cfg rc=$?
