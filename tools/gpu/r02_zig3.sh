python -m pytest tests/test_gpu_parity.py tests/test_gpu_probgen.py tests/test_gpu_multidevice.py -x -q -k "gauss or normal or probgen or generate or band" 2>&1 | tail -2
SKL_ZIG_PROBE=1 python tools/prof_gauss_gen.py
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"zig_write|zig_spec" -c 2 python tools/prof_gauss_gen.py 2>&1 | grep -E "^  zig_|duration|inst_exec" | cut -c1-100
