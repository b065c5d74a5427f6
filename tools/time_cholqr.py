"""Reduced-solve timing: CholeskyQR2 path (skl_cqr_solve_async) against the
Householder path (skl_qr_solve_async) on the sketched shapes of the BASELINE
configs; CUDA events on the launching stream, median of 20 after warm-up."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_14309_b200 import _native  # noqa: E402
from paper_2409_14309_b200._device import current_stream  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


shapes = [(800, 200), (2048, 256), (2048, 511), (8192, 511)] if len(sys.argv) < 2 else \
    [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
flags = torch.zeros(2, dtype=torch.float64, pin_memory=True)
for d, n in shapes:
    rng = np.random.default_rng(0)
    SA = torch.from_numpy(np.asfortranarray(rng.standard_normal((d, n)))).cuda().t().contiguous().t()
    Sb = torch.from_numpy(rng.standard_normal(d)).cuda()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    st = current_stream()
    base = flags.data_ptr()

    def cqr():
        _native.call("skl_cqr_solve_async", _native.ptr(SA), d, _native.ptr(Sb), d, n,
                     _native.ptr(x), base, base + 8, st)

    def hh():
        _native.call("skl_qr_solve_async", _native.ptr(SA), d, _native.ptr(Sb), d, n,
                     _native.ptr(x), None, n, None, d, base, base + 8, st)

    t_c = timed(cqr)
    xc = x.clone()
    t_h = timed(hh)
    xh = x.clone()
    print(json.dumps({"d": d, "n": n, "cholqr_ms": round(t_c, 4), "householder_ms": round(t_h, 4),
                      "x_rel_diff": float((xc - xh).norm() / xh.norm()),
                      "flag": int(flags.view(torch.int64)[0])}), flush=True)
