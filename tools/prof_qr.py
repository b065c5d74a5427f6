"""Profiling driver for the reduced solve: QR + back-solve of a d x n
sketched system (default: config 4's 8192 x 1024, and config 2's 2048 x 256).

The GPU is kept busy for ~0.5 s before timing (clocks ramp up under load),
then `reps` solves are timed one by one with CUDA events; the median and the
SM clock read through NVML right after are printed."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2409_14309_b200.linalg import qr_solve_device, reduced_solve_device  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
# 4th argument "cholqr": the path sketch_and_apply takes (CholeskyQR2 + CSNE
# when eligible); default: the Householder factorisation
if len(sys.argv) > 4 and sys.argv[4] == "cholqr":
    def qr_solve_device(M, ld, y, d, n):  # noqa: F811
        return reduced_solve_device(M, ld, y, d, n), None, None
warm_s = float(__import__("os").environ.get("SKL_PROF_WARM_S", "0.5"))
M = torch.randn((n, d), dtype=torch.float64, device="cuda").t()
y = torch.randn((d,), dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
while time.perf_counter() - t0 < warm_s:
    qr_solve_device(M, d, y, d, n)
    torch.cuda.synchronize()
ts = []
for _ in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    qr_solve_device(M, d, y, d, n)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
clk = ""
try:
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    clk = f" sm_clock {pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)} MHz"
except Exception:  # noqa: BLE001 -- the clock is informational
    pass
print(f"qr_solve {d}x{n}: {statistics.median(ts):.3f} ms (median of {reps}, min "
      f"{min(ts):.3f}){clk}")
