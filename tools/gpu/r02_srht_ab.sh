timeout 200 python tools/time_srht.py ld66 20 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "srht" 2>&1 | tail -1
export SKL_NVCC_DEFINES=-DSKL_SR2_LD=65
python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)" 2>&1 | tail -1
timeout 200 python tools/time_srht.py ld65 20 2>&1 | tail -1
