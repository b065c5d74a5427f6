set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multidevice.py tests/test_gpu_slots.py -x -q 2>&1 | tail -5
python tools/time_multidevice.py > gpurun_out/r02_multidevice.json; cat gpurun_out/r02_multidevice.json
