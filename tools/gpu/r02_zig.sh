python -m pytest tests/test_gpu_parity.py tests/test_gpu_probgen.py tests/test_gpu_multidevice.py -x -q -k "gauss or normal or probgen or generate or band" 2>&1 | tail -2
python tools/prof_gauss_gen.py
