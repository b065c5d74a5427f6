"""Profiling driver: CountSketch operator construction on the device (device
RNG + register-owned plan) for config 2 (2^20 rows, d = 2048), repeated."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402

m, d = 1 << 20, 2048
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(reps):
    E.clear_operator_cache()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=7), m)
    op.device_plan()
    torch.cuda.synchronize()
    print(f"build {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms")
