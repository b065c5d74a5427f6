for ch in 0 4096 6144 2048; do SKL_OWNED_CHUNK=$ch timeout 120 python tools/time_sketch.py 2 2>&1 | tail -1; done
for st in 2 3; do SKL_OWNED_STAGES=$st timeout 120 python tools/time_sketch.py 2 2>&1 | tail -1; done
