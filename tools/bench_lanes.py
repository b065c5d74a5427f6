"""Dense CountSketch with d > 2048 (lane-list plan, shared-memory bucket sums):
kernel time and HBM fraction for a 2^20 x n fp64 A at several d."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200.sketch import _countsketch_dense_device  # noqa: E402

PEAK = 6451.2
m = 1 << 20
for n, d in ((256, 2048), (256, 4096), (256, 8192), (1024, 8192), (256, 16384)):
    A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    b = torch.randn((m,), dtype=torch.float64, device="cuda")
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=1), m)
    plan = op.device_plan()
    for _ in range(2):
        _countsketch_dense_device(op, A, m, n, b=b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        _countsketch_dense_device(op, A, m, n, b=b)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    gbs = 8 * m * (n + 1) / ms / 1e6
    print(json.dumps({"n": n, "d": d, "plan": plan.kind, "ms": round(ms, 4), "gbs": round(gbs, 1),
                      "frac": round(gbs / PEAK, 3)}))
    del A, op
    torch.cuda.empty_cache()
