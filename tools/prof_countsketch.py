"""Profiling driver: a few launches of the dense CountSketch kernel on the
config-2 shape (2^20 x 256 fp64, d = 2048), device-resident inputs.
Used under ncu (see profiles/README.md)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from paper_2409_14309_b200.sketch import _countsketch_dense_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = W.config(cfg, kind="countsketch")
m, n, d = c.m, c.n, c.d
A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
b = torch.randn((m,), dtype=torch.float64, device="cuda")
op = E.build_sketch(E.SketchSpec("countsketch", d, seed=1), m)
for _ in range(reps):
    _countsketch_dense_device(op, A, m, n, b=b)
torch.cuda.synchronize()
print("ok")
