"""SAP (sketch-and-precondition + LSQR) on a full-size config, one GPU:
per-iteration GEMV timings against the HBM roofline and whole-solve time.

    python tools/bench_sap.py [cfg]   (default 2)
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native, workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = W.config(cfg)
A, b, _ = W.make_problem(c, backend="torch")
m, n = c.m, c.n
lda = int(A.stride(1))
prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
spec = E.SketchSpec(c.kind, 1, seed=W.SEED)
opts = E.SolverOptions(d_factor=c.d / c.n)
E.solve(prob, "sap", spec, opts)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = E.solve(prob, "sap", spec, opts)
torch.cuda.synchronize()
t_sap = time.perf_counter() - t0

# kernel timings of one iteration's two passes over A
st = torch.cuda.current_stream().cuda_stream
y = torch.randn(n, dtype=torch.float64, device="cuda")
u = torch.randn(m, dtype=torch.float64, device="cuda")
u2 = torch.empty_like(u)
z = torch.empty(n, dtype=torch.float64, device="cuda")
sc = torch.zeros(2, dtype=torch.float64, device="cuda")
work = torch.empty(int(_native.lib().skl_lsqr_work_size(m, n)), dtype=torch.float64, device="cuda")
cnt = torch.zeros(int(_native.lib().skl_lsqr_counter_size(n)), dtype=torch.int32, device="cuda")


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    bb.record()
    torch.cuda.synchronize()
    return a.elapsed_time(bb) / reps


tn = timed(lambda: _native.call("skl_lsqr_gemv_n", A.data_ptr(), m, n, lda, y.data_ptr(), 1.0,
                                0.5, u.data_ptr(), u2.data_ptr(), sc.data_ptr(), work.data_ptr(),
                                cnt.data_ptr(), st))
tt = timed(lambda: _native.call("skl_lsqr_gemv_t", A.data_ptr(), m, n, lda, u2.data_ptr(), 2.0,
                                u.data_ptr(), z.data_ptr(), work.data_ptr(), cnt.data_ptr(), st))
gb = 8.0 * m * n / 1e9
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())[
    "hbm_gbs"] if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6451.2
print(json.dumps({
    "config": cfg, "m": m, "n": n, "d": c.d, "kind": c.kind,
    "sap": {"ms_per_solve": round(t_sap * 1e3, 2), "iterations": res.iterations,
            "termination": res.termination, "residual": res.residual_norm},
    "gemv_n_ms": round(tn, 4), "gemv_n_gbs": round(gb / tn * 1e3, 1),
    "gemv_n_frac": round(gb / tn * 1e3 / peak, 3),
    "gemv_t_ms": round(tt, 4), "gemv_t_gbs": round(gb / tt * 1e3, 1),
    "gemv_t_frac": round(gb / tt * 1e3 / peak, 3)}))
