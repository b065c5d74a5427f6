"""Gaussian apply GEMM at config 3: G (2048 x 262144, row-major) times A
(262144 x 512, column-major) through skl_gemm_f64, median of `reps` by CUDA
events, with cuBLAS DGEMM (torch) on the same operands beside it and the
result's relative difference from a result saved by an earlier run (build
variants on one box).  Usage: python tools/time_gemm.py TAG [reps]"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2409_14309_b200 import _native  # noqa: E402

tag = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
d, m, n = 2048, 262144, 512
g = torch.Generator(device="cuda").manual_seed(3)
G = torch.randn((d, m), dtype=torch.float64, device="cuda", generator=g)
A = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g).t()
C = torch.empty((n, d), dtype=torch.float64, device="cuda").t()


def ours():
    _native.call("skl_gemm_f64", G.data_ptr(), m, A.data_ptr(), m, C.data_ptr(), d, d, n, m, 0,
                 torch.cuda.current_stream().cuda_stream)


def timed(fn):
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


t = timed(ours)
base = Path("/tmp/gemm_ref.pt")
diff = None
if base.exists():
    ref = torch.load(base)
    diff = float((C - ref).norm() / ref.norm())
else:
    torch.save(C.clone(), base)
rec = {"tag": tag, "defines": os.environ.get("SKL_NVCC_DEFINES", ""), "ms": round(t, 3),
       "tflops": round(2 * d * n * m / t / 1e9, 2), "rel_diff_vs_first": diff}
if "--cublas" in sys.argv:
    tc = timed(lambda: torch.mm(G, A))
    rec.update(cublas_ms=round(tc, 3), cublas_tflops=round(2 * d * n * m / tc / 1e9, 2))
print(json.dumps(rec), flush=True)
