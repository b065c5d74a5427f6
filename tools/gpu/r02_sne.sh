timeout 600 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -3
timeout 300 python tools/time_cholqr.py 800x200 2048x256 2048x600 8192x1024 2>&1 | tail -4
SKL_NO_PDL=1 timeout 300 python tools/prof_cqr_kernels.py 8192 1024 2>&1 | tail -18
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k: d['solve'][k] for k in ('solves_per_sec','batched_solves_per_sec','qr_solve_ms','householder_qr_solve_ms','qr_path')})"
