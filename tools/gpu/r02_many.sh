timeout 600 python -m pytest tests/test_gpu_api_properties.py -q -k "solve_many" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --no-e2e > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
tail -2 gpurun_out/r02_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r02_bench.out').read().strip().splitlines()[-1]); print(d['value'], {k: d['solve'][k] for k in ('solves_per_sec','ms_per_solve','batched_solves_per_sec','batched_ms_per_solve','qr_solve_ms')})"
