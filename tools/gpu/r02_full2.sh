mkdir -p gpurun_out
SKL_PARITY_REPORT=gpurun_out/r02_parity_fullsize.jsonl timeout 2000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -8
timeout 600 python bench.py > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r02_bench.out').read().strip().splitlines()[-1]); print(d['value'], d['solve'])"
