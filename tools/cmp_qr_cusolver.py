"""Reduced solve: skl_qr_solve against cuSOLVER (torch.linalg.qr = geqrf +
orgqr, then Q^T y and a triangular solve) on the sketched shapes of every
BASELINE config.  Both timed by CUDA events on the current stream, median
of `reps` after warm-up.  Prints one JSON line per shape."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2409_14309_b200.linalg import qr_solve_device  # noqa: E402

SHAPES = [(800, 200), (2048, 256), (2048, 512), (8192, 1024)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for d, n in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(d + n)
    M = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g).t()
    y = torch.randn((d,), dtype=torch.float64, device="cuda", generator=g)
    x_ours = qr_solve_device(M, d, y, d, n)[0]

    def cus():
        Q, R = torch.linalg.qr(M, mode="reduced")
        return torch.linalg.solve_triangular(R, (Q.t() @ y).unsqueeze(1), upper=True)

    def cus_r_only():
        # geqrf alone (R in the upper triangle, Householder vectors below)
        return torch.geqrf(M)

    x_cus = cus().squeeze(1)
    rel = float((x_ours - x_cus).norm() / x_cus.norm())
    t_ours = timed(lambda: qr_solve_device(M, d, y, d, n))
    t_cus = timed(cus)
    t_geqrf = timed(cus_r_only)
    print(json.dumps({"d": d, "n": n, "skl_qr_solve_ms": round(t_ours, 4),
                      "cusolver_qr_solve_ms": round(t_cus, 4),
                      "cusolver_geqrf_only_ms": round(t_geqrf, 4),
                      "speedup_vs_cusolver": round(t_cus / t_ours, 3),
                      "x_rel_diff": rel}), flush=True)
