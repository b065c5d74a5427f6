timeout 900 python -m pytest tests -m gpu -q -x -k "lsqr or sap or LSQR or SAP" 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d['solve'][k] for k in ('sap_ms_per_solve','solves_per_sec')})"
SKL_LSQR_BLOCK_SOLVES=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d['solve'][k] for k in ('sap_ms_per_solve','solves_per_sec')})"
