import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from test_gpu_cholqr import system, cqr, oracle_x
cases = [(2456, 1030, k) for k in (10.0, 1e4, 1e6, 5e7)] + [(2456, 1024, 5e7), (2456, 1000, 5e7), (4096, 1030, 5e7),
         (2464, 1030, 5e7), (2048, 1030, 5e7), (3000, 1030, 5e7), (2456, 700, 5e7), (2456, 530, 5e7), (2456, 510, 5e7)]
for (d, n, kappa) in cases:
    SA, Sb = system(d, n, kappa=kappa, seed=7 + n)
    x, fb = cqr(SA, Sb)
    want = oracle_x(SA, Sb)
    rs, rw = np.linalg.norm(SA @ x - Sb), np.linalg.norm(SA @ want - Sb)
    print(f"{d}x{n} kappa {kappa:.0e} fb {fb} resid_excess {rs / rw - 1:.2e} xerr {np.linalg.norm(x - want) / np.linalg.norm(want):.2e}", flush=True)
