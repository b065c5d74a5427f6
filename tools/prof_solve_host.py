"""Host-side cost of one sketch-and-apply solve() on device data (config 2):
cProfile of 200 warm solves, top functions by own time."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402

c = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
A, b, _ = W.make_problem(c, backend="torch")
A = E.SparseMatrix.from_scipy(A) if c.gen == "csr" else E.DenseMatrix(A)
prob = E.LeastSquaresProblem(A, E.Vector(b))
spec, opts = E.SketchSpec(c.kind, 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n)
for _ in range(5):
    E.solve(prob, "saa", spec, opts)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    E.solve(prob, "saa", spec, opts)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
pstats.Stats(pr).sort_stats("cumtime").print_stats(14)
