"""Where the time of one SAA solve goes (config 2 shape, device-resident A):
the public solve() against its stages timed alone (CUDA events, warm), and
the host time one solve() call takes to enqueue."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from paper_2409_14309_b200.linalg import qr_solve_device, qr_solve_device_async  # noqa: E402
from paper_2409_14309_b200.sketch import _countsketch_dense_device  # noqa: E402
from paper_2409_14309_b200.solvers import _residual_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = W.config(cfg, kind="countsketch")
A, b, _ = W.make_problem(c, backend="torch")
prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
spec, opts = E.SketchSpec("countsketch", 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n)
for _ in range(3):
    E.solve(prob, "saa", spec, opts)
torch.cuda.synchronize()


def wall(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


def events(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


op = E.build_sketch(E.solvers._operator_spec(spec, "saa", c.m, c.n, opts.d_factor), c.m)
SA, Sb = _countsketch_dense_device(op, A, int(A.stride(1)), c.n, b=b)
x, _, _ = qr_solve_device(SA, c.d, Sb, c.d, c.n)
out = {
    "solve_wall_ms": wall(lambda: E.solve(prob, "saa", spec, opts)),
    "sketch_ms": events(lambda: _countsketch_dense_device(op, A, int(A.stride(1)), c.n, b=b)),
    "qr_ms": events(lambda: qr_solve_device_async(SA, c.d, Sb, c.d, c.n)),
    "householder_qr_ms": events(lambda: qr_solve_device(SA, c.d, Sb, c.d, c.n)),
    "solve_events_ms": events(lambda: E.solve(prob, "saa", spec, opts)),
    "residual_wall_ms": wall(lambda: _residual_device(prob.A, A, int(A.stride(1)), b, x)),
}
t0 = time.perf_counter()
for _ in range(20):
    _countsketch_dense_device(op, A, int(A.stride(1)), c.n, b=b)
out["sketch_enqueue_us"] = (time.perf_counter() - t0) / 20 * 1e6
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    qr_solve_device_async(SA, c.d, Sb, c.d, c.n)
out["qr_enqueue_us"] = (time.perf_counter() - t0) / 20 * 1e6
torch.cuda.synchronize()
print({k: round(v, 4) for k, v in out.items()})

# cold solves: the operator (device draws + device plan) rebuilt every solve,
# as the reference rebuilds it (solvers.py:279 -> sketch.py:84)
def cold_solve():
    E.clear_operator_cache()
    E.solve(prob, "saa", spec, opts)


def cold_build():
    E.clear_operator_cache()
    o = E.build_sketch(E.solvers._operator_spec(spec, "saa", c.m, c.n, opts.d_factor), c.m)
    o.device_plan()


print({"cold_solve_wall_ms": round(wall(cold_solve), 4),
       "cold_build_wall_ms": round(wall(cold_build), 4)})
