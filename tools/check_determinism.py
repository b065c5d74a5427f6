"""Run the same SAA / SAP solves many times in one process and check that
every result is bitwise identical (the device paths fix every reduction
order, so any difference means a race).  Usage: check_determinism.py [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bad = 0
for cfg, m, n, d, method in [(2, 1 << 14, 256, 2048, "saa"), (1, 20000, 200, 800, "saa"),
                             (2, 1 << 14, 256, 2048, "sap"), (3, 1 << 14, 512, 2048, "saa")]:
    c = W.config(cfg, m=m, n=n, d=d)
    A, b, _ = W.make_problem(c)
    kind = "countsketch" if cfg != 3 else "gaussian"
    for host in (True, False):
        Ad = A if host else torch.from_numpy(np.asfortranarray(A)).cuda()
        bd = b if host else torch.from_numpy(b).cuda()
        prob = E.LeastSquaresProblem(E.DenseMatrix(Ad), E.Vector(bd))
        spec = E.SketchSpec(kind, 1, seed=W.SEED)
        opts = E.SolverOptions(d_factor=d / n)
        first = None
        for r in range(reps):
            res = E.solve(prob, method, spec, opts)
            x = res.x.data if isinstance(res.x.data, np.ndarray) else res.x.data.cpu().numpy()
            if first is None:
                first = (x.copy(), res.residual_norm)
            elif not (np.array_equal(x, first[0]) and res.residual_norm == first[1]):
                bad += 1
                print(f"MISMATCH cfg{cfg} {method} host={host} rep {r}: "
                      f"max|dx|={np.max(np.abs(x - first[0])):.3e}", flush=True)
        print(f"cfg{cfg} {method} host={host}: {reps} solves checked", flush=True)
print("determinism:", "FAIL" if bad else "ok", bad)
