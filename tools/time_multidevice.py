"""Cost pieces of the multi-device paths, measured on ONE GPU.

* config 3's Gaussian operator: the one-device generation of all of G
  against one band of an N-device banded generation (what each device does
  on an N-GPU node) and the band-to-block exchange;
* solve() over an emulated device list (devices=(0,)*N): the shard / reduce
  overhead of the N-shard logic when every shard runs on the same GPU (not a
  scaling number: the work is not spread)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from paper_2409_14309_b200.distributed import shard_rows  # noqa: E402
from paper_2409_14309_b200.multidevice import gaussian_column_blocks  # noqa: E402


def wall(fn, reps=3):
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


out = {}
c3 = W.config(3)
spec3 = E.SketchSpec("gaussian", c3.d, seed=7)


def full_g():
    op = E.build_sketch(spec3, c3.m)
    E.clear_operator_cache()
    op.device_gaussian()


out["cfg3_full_G_one_device_ms"] = round(wall(full_g), 2)
for world in (2, 4, 8):
    spans = [shard_rows(c3.m, world, k) for k in range(world)]
    op = E.build_sketch(spec3, c3.m)
    E.clear_operator_cache()
    t = wall(lambda: gaussian_column_blocks(op, (0,) * world, spans), reps=2)
    out[f"cfg3_banded_{world}_bands_on_one_gpu_ms"] = round(t, 2)
    out[f"cfg3_banded_{world}_per_device_estimate_ms"] = round(t / world, 2)

for cfg in (2,):
    c = W.config(cfg, kind="countsketch")
    A, b, _ = W.make_problem(c, backend="torch")
    prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
    spec = E.SketchSpec("countsketch", 1, seed=W.SEED)
    for world in (1, 2, 4, 8):
        opts = E.SolverOptions(d_factor=c.d / c.n, devices=(0,) * world if world > 1 else None)
        E.solve(prob, "saa", spec, opts)
        out[f"cfg{cfg}_solve_emulated_{world}_shards_ms"] = round(
            wall(lambda: E.solve(prob, "saa", spec, opts), reps=5), 3)
print(json.dumps(out))
