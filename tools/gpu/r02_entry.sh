timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
timeout 120 python bench.py --gpus 2 --steps 2 --warmup 3 > /dev/null 2> gpurun_out/g2.err; echo "gpus2 rc=$?"; tail -1 gpurun_out/g2.err
