mkdir -p gpurun_out
SKL_NVCC_DEFINES=-DSKL_ZIG_RING_WRITE python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:zig_write -c 1 -o gpurun_out/r02_zig_write_ring python tools/prof_gauss_gen.py > /dev/null 2>&1
ncu -i gpurun_out/r02_zig_write_ring.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_zig_write_ring_sass.csv 2>&1
echo done
