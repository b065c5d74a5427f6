"""Compare the register-owned CountSketch kernel with the lane-list kernel:
bitwise equality and device time on the config-2 shape (2^20 x 256, d=2048)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
d = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
chunks = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2048, 4096]
warps = 16 if d > 1024 else 8
torch.manual_seed(0)
A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
b = torch.randn((m,), dtype=torch.float64, device="cuda")
op = E.build_sketch(E.SketchSpec("countsketch", d, seed=1), m)
st = torch.cuda.current_stream().cuda_stream


def bench(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gb = (m * (n + 1) * 8) / 1e9
lanes, off, mx = _native.countsketch_plan(op.rows, op.signs, d, 2048, warps)
L, O = torch.from_numpy(lanes).cuda(), torch.from_numpy(off).cuda()
SA0 = torch.empty((n, d), dtype=torch.float64, device="cuda")
Sb0 = torch.empty((d,), dtype=torch.float64, device="cuda")
f0 = lambda: _native.call("skl_countsketch_dense", A.data_ptr(), m, n, m, b.data_ptr(), L.data_ptr(),
                          O.data_ptr(), mx, d, 2048, warps, SA0.data_ptr(), d, Sb0.data_ptr(), 0, 0, st)
t = bench(f0)
print(f"lane-list chunk 2048: {t:.3f} ms  {gb / t * 1e3:.0f} GB/s  plan {lanes.nbytes / m:.2f} B/row")
for ch in chunks:
    t0 = time.perf_counter()
    lo, oo, mo = _native.countsketch_plan_owned(op.rows, op.signs, d, ch, warps)
    tp = time.perf_counter() - t0
    L2, O2 = torch.from_numpy(lo.view(np.int16)).cuda(), torch.from_numpy(oo).cuda()
    SA1 = torch.empty((n, d), dtype=torch.float64, device="cuda")
    Sb1 = torch.empty((d,), dtype=torch.float64, device="cuda")
    f1 = lambda: _native.call("skl_countsketch_dense_owned", A.data_ptr(), m, n, m, b.data_ptr(),
                              L2.data_ptr(), O2.data_ptr(), mo, d, ch, warps, SA1.data_ptr(), d,
                              Sb1.data_ptr(), 0, 0, st)
    t = bench(f1)
    same = torch.equal(SA0, SA1) and torch.equal(Sb0, Sb1)
    util = m / (lo.size / 1.0)
    print(f"owned chunk {ch}: {t:.3f} ms  {gb / t * 1e3:.0f} GB/s  bitwise={same}  "
          f"plan {lo.nbytes / m:.2f} B/row  util {util:.2f}  plan build {tp * 1e3:.0f} ms")
