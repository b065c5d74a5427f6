"""Warm per-kernel times of the CholeskyQR2 reduced solve (torch.profiler,
CUDA activity), averaged over `reps` solves of a d x n system.  Run with
SKL_NO_PDL=1: with programmatic dependent launch a kernel's recorded span
starts while its predecessor still runs.  Usage: prof_cqr_kernels.py d n [reps] [kappa]
(kappa: log-spaced singular values, e.g. 1e8 = config 2; default a Gaussian SA)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_14309_b200.linalg import reduced_solve_device  # noqa: E402

d, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
kappa = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
if kappa > 0:
    U, _ = torch.linalg.qr(torch.randn((d, n), dtype=torch.float64, device="cuda"))
    V, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device="cuda"))
    sv = torch.logspace(0, -torch.log10(torch.tensor(kappa)).item(), n, dtype=torch.float64, device="cuda")
    M = ((U * sv) @ V.t()).t().contiguous().t()
else:
    M = torch.randn((n, d), dtype=torch.float64, device="cuda").t()
y = torch.randn((d,), dtype=torch.float64, device="cuda")
for _ in range(20):
    reduced_solve_device(M, d, y, d, n)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        reduced_solve_device(M, d, y, d, n)
    torch.cuda.synchronize()
rows = [(e.key, e.device_time_total / reps, e.count / reps) for e in prof.key_averages()
        if e.device_time_total > 0]
tot = sum(r[1] for r in rows)
print(f"{d}x{n}: kernel total {tot:.1f} us per solve")
for k, t, c in sorted(rows, key=lambda r: -r[1]):
    print(f"  {t:8.1f} us  x{c:4.1f}  {k[:90]}")
