import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from test_gpu_cholqr import system, cqr, oracle_x
for (d, n) in [(2048, 256), (2456, 1030), (8192, 1024), (3000, 700)]:
    for kappa in [5e7, 1e8, 2e8, 3e8, 6e8]:
        SA, Sb = system(d, n, kappa=kappa, seed=7 + n)
        x, fb = cqr(SA, Sb)
        want = oracle_x(SA, Sb)
        r = np.linalg.qr(SA, mode="r"); dg = np.abs(np.diag(r)); ratio = dg.max() / dg.min()
        rs, rw = np.linalg.norm(SA @ x - Sb), np.linalg.norm(SA @ want - Sb)
        print(f"{d}x{n} kappa {kappa:.0e} ratio {ratio:.2e} fb {fb} resid_excess {rs / rw - 1:.2e} xerr {np.linalg.norm(x - want) / np.linalg.norm(want):.2e}", flush=True)
