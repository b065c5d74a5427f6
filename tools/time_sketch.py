"""CUDA-event time of the config-2 dense CountSketch apply S[A|b] (device
inputs, 2 GiB > L2), median of 20 -- for A/B runs of build knobs."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from paper_2409_14309_b200.sketch import _countsketch_dense_device  # noqa: E402

c = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2, kind="countsketch")
m, n, d = c.m, c.n, c.d
A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
b = torch.randn((m,), dtype=torch.float64, device="cuda")
op = E.build_sketch(E.SketchSpec("countsketch", d, seed=1), m)
for _ in range(5):
    _countsketch_dense_device(op, A, m, n, b=b)
ts = []
for _ in range(20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _countsketch_dense_device(op, A, m, n, b=b)
    e.record()
    e.synchronize()
    ts.append(s.elapsed_time(e))
ms = statistics.median(ts)
print(f"cfg {c.cfg} chunk {op.device_plan().chunk if hasattr(op.device_plan(), 'chunk') else '?'}: "
      f"{ms:.4f} ms  {8 * m * (n + 1) / ms / 1e6:.0f} GB/s")
