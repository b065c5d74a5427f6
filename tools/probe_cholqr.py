"""Per-phase timeline of the cluster Cholesky (build with
SKL_NVCC_DEFINES=-DSKL_CQR_PROBE): one warm CholeskyQR2 solve of a d x n
system, then per CTA and step the ns since the kernel's first timestamp."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_14309_b200 import _native  # noqa: E402
from paper_2409_14309_b200.linalg import reduced_solve_device  # noqa: E402

d, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048x256").split("x"))
rng = np.random.default_rng(0)
SA = torch.from_numpy(np.asfortranarray(rng.standard_normal((d, n)))).cuda().t().contiguous().t()
Sb = torch.from_numpy(rng.standard_normal(d)).cuda()
for _ in range(3):
    reduced_solve_device(SA, d, Sb, d, n)
buf = np.zeros((2, 16, 72), dtype=np.int64)
fn = _native.lib().skl_cqr_probe_dump
fn.argtypes = [ctypes.c_void_p]
fn(buf.ctypes.data)
nb = (n + 1 + 31) // 32
for it in range(2):
    t0 = min(buf[it, j, 0] for j in range(nb))
    print(f"--- cholesky {it + 1}: total {(max(buf[it, j, 70] for j in range(nb)) - t0) / 1e3:.1f} us")
    for j in range(nb):
        row = buf[it, j]
        steps = " ".join(f"[{(row[2 + 4 * k] - t0) / 1e3:.1f} {(row[3 + 4 * k] - t0) / 1e3:.1f} "
                         f"{(row[4 + 4 * k] - t0) / 1e3:.1f} {(row[5 + 4 * k] - t0) / 1e3:.1f}]"
                         for k in range(nb - 1))
        print(f"cta {j:2d} start {(row[0] - t0) / 1e3:.1f} loaded {(row[1] - t0) / 1e3:.1f} "
              f"end {(row[70] - t0) / 1e3:.1f} | {steps}")
