timeout 300 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_fullsize.py -q -k "cholqr or cfg2 or cfg5" 2>&1 | tail -2
timeout 200 python tools/time_cholqr.py 800x200 2048x256 2048x511 8192x511 2>&1 | tail -4
timeout 600 python bench.py --steps 20 > gpurun_out/r02_bench.out 2> gpurun_out/r02_bench.err; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r02_bench.out').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], {k: d['solve'][k] for k in ('solves_per_sec','ms_per_solve','qr_solve_ms','qr_path','householder_qr_solve_ms','solves_per_sec_cold')})"
