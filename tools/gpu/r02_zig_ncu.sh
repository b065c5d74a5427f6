mkdir -p gpurun_out
python tools/prof_gauss_gen.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_zig_launches.csv python tools/prof_gauss_gen.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:zig_spec -c 1 -o gpurun_out/r02_zig_spec python tools/prof_gauss_gen.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:zig_write -c 1 -o gpurun_out/r02_zig_write python tools/prof_gauss_gen.py > /dev/null 2>&1
echo done
