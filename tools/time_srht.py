"""SRHT apply at config 5 (2^23 x 256, d = 2048): median kernel time by CUDA
events over `reps` launches, and the result's relative difference from a
saved earlier run (for comparing build variants on one box).
Usage: python tools/time_srht.py TAG [reps] [m_log2] [n]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200.sketch import _srht_device  # noqa: E402

tag = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
m = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 23)
n = int(sys.argv[4]) if len(sys.argv) > 4 else 256
d = 2048
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g).t()
op = E.build_sketch(E.SketchSpec("srht", d, seed=1), m)
SA = _srht_device(op, A, m, n)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _srht_device(op, A, m, n)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
ms = ts[len(ts) // 2]
base = Path(f"/tmp/srht_ref_{m}_{n}.pt")
diff = None
if base.exists():
    ref = torch.load(base)
    diff = float((SA - ref).norm() / ref.norm())
else:
    torch.save(SA, base)
print(json.dumps({"tag": tag, "defines": os.environ.get("SKL_NVCC_DEFINES", ""), "m": m, "n": n,
                  "ms": round(ms, 4), "tbs": round(8 * m * n / ms / 1e9, 3),
                  "rel_diff_vs_first": diff}), flush=True)
