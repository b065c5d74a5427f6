"""Profiling driver: a few launches of one sketch kernel on device-resident
inputs.  Usage: python tools/prof_kernels.py {srht|csr|gauss|resid} [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native, workloads as W  # noqa: E402
from paper_2409_14309_b200.sketch import (  # noqa: E402
    _countsketch_csr_device,
    _gaussian_device,
    _srht_device,
)

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "srht":
    m, n, d = 1 << 23, 256, 2048  # config 5
    A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    op = E.build_sketch(E.SketchSpec("srht", d, seed=1), m)
    for _ in range(reps):
        _srht_device(op, A, m, n)
elif which == "csr":
    c = W.config(4)
    A, b, _ = W.make_problem(c, backend="torch")
    Ac = E.SparseMatrix.from_scipy(A)
    op = E.build_sketch(E.SketchSpec("countsketch", c.d, seed=1), c.m)
    for _ in range(reps):
        _countsketch_csr_device(op, Ac)
elif which == "gauss":
    m, n, d = 262144, 512, 2048
    A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    op = E.build_sketch(E.SketchSpec("gaussian", d, seed=1), m)
    op.device_gaussian()
    for _ in range(reps):
        _gaussian_device(op, A, m, n)
elif which == "resid":
    m, n = 1 << 20, 256
    A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    x = torch.randn((n,), dtype=torch.float64, device="cuda")
    b = torch.randn((m,), dtype=torch.float64, device="cuda")
    import numpy as np

    out = np.zeros(1)
    for _ in range(reps):
        _native.call("skl_residual_dense", A.data_ptr(), m, n, m, x.data_ptr(), b.data_ptr(),
                     out.ctypes.data, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", which)
