"""Kernel-level breakdown of one warm solve() (method argv[2], default saa) for a BASELINE config
(torch.profiler CUDA activity: every kernel and copy of the solve)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
method = sys.argv[2] if len(sys.argv) > 2 else "saa"
c = W.config(cfg)
A, b, _ = W.make_problem(c, backend="torch")
if c.gen == "csr":
    A = E.SparseMatrix.from_scipy(A)
else:
    A = E.DenseMatrix(A)
prob = E.LeastSquaresProblem(A=A, b=E.Vector(b))
spec = E.SketchSpec(c.kind, 1, seed=W.SEED)
opts = E.SolverOptions(d_factor=c.d / c.n)
for _ in range(2):
    E.solve(prob, method, spec, opts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    E.solve(prob, method, spec, opts)
    torch.cuda.synchronize()
rows = [(e.key, e.device_time_total, e.count) for e in prof.key_averages() if e.device_time_total > 0]
tot = sum(r[1] for r in rows)
for k, t, n in sorted(rows, key=lambda r: -r[1])[:25]:
    print(f"{t / 1e3:9.3f} ms  x{n:<3d} {k[:70]}")
print(f"{tot / 1e3:9.3f} ms  total device time (PDL-chained kernels include their early start)")
