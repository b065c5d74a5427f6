"""Sparse sign embedding apply (s = 8) on the config-2 shape, one GPU:
S [A | b] time and algorithmic GB/s (bytes of A and b)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200.sketch import _countsketch_dense_device  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
d = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
s = int(sys.argv[4]) if len(sys.argv) > 4 else 8
A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
b = torch.randn((m,), dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
op = E.build_sketch(E.SketchSpec("sparsesign", d, seed=1, sparsity=s), m)
t1 = time.perf_counter()
plan = op.device_plan()
torch.cuda.synchronize()
t2 = time.perf_counter()
for _ in range(2):
    _countsketch_dense_device(op, A, m, n, b=b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 10
for _ in range(reps):
    _countsketch_dense_device(op, A, m, n, b=b)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = 8.0 * m * (n + 1) / 1e9
print(json.dumps({"m": m, "n": n, "d": d, "s": s, "apply_ms": round(ms, 4),
                  "gbs": round(gb / ms * 1e3, 1), "draws_ms": round((t1 - t0) * 1e3, 1),
                  "plan_ms": round((t2 - t1) * 1e3, 1), "chunk": plan.chunk}))
