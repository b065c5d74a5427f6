"""Time the Gaussian operator generation (config 3: 2048 x 262144) stage by stage."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2409_14309_b200 as E
for rep in range(2):
    E.clear_operator_cache()
    op = E.build_sketch(E.SketchSpec("gaussian", 2048, seed=rep), 262144)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.device_gaussian()
    torch.cuda.synchronize()
    print(f"generate G: {(time.perf_counter() - t0) * 1e3:.2f} ms")
