mkdir -p gpurun_out
SKL_PARITY_REPORT=gpurun_out/r02_parity_fullsize.jsonl timeout 2000 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6
