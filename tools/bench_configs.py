"""Per-config kernel and solve timings on one GPU (all five BASELINE configs).

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--reps 10]

For every config: the sketch kernel(s) on device-resident inputs (CUDA
events, median of reps), algorithmic GB/s (or fp64 TFLOP/s for the
Gaussian GEMM, beside cuBLAS DGEMM via torch.matmul on the same operands
as the measured fp64 peak), the reduced QR solve, and full SAA solves/sec
through the public API.  One JSON line per config on stdout.  Config 5
runs both SRHT and CountSketch on the same 16 GiB matrix.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from paper_2409_14309_b200.linalg import (cholqr_enabled, qr_solve_device,  # noqa: E402
                                          reduced_solve_device)
from paper_2409_14309_b200.sketch import (  # noqa: E402
    _countsketch_csr_device,
    _countsketch_dense_device,
    _gaussian_device,
    _srht_device,
)

PEAK_HBM = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())[
    "hbm_gbs"] if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def timed_graph(fn, reps):
    """Device time of fn: captured once in a CUDA graph and replayed between
    CUDA events, so small kernels are not timed behind the host's launch
    overhead.  Falls back to timed() when the call cannot be captured."""
    try:
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
    except Exception:  # noqa: BLE001 - capture unsupported: plain timing
        torch.cuda.synchronize()
        return timed(fn, reps), False
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), True


def solve_rate(A, b, kind, d, n, reps=3):
    prob = E.LeastSquaresProblem(A=A, b=E.Vector(b))
    spec = E.SketchSpec(kind, 1, seed=W.SEED)
    opts = E.SolverOptions(d_factor=d / n)
    E.solve(prob, "saa", spec, opts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        res = E.solve(prob, "saa", spec, opts)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return {"solves_per_sec": round(1 / dt, 3), "ms_per_solve": round(dt * 1e3, 3),
            "residual": res.residual_norm}


def run(cfg_id: int, reps: int):
    c = W.config(cfg_id)
    out = {"config": cfg_id, "m": c.m, "n": c.n, "d": c.d, "kind": c.kind}
    A, b, _ = W.make_problem(c, backend="torch")
    if c.gen == "csr":
        Ac = E.SparseMatrix.from_scipy(A)
        nnz = Ac.nnz
        op = E.build_sketch(E.SketchSpec("countsketch", c.d, seed=1), c.m)
        op.device_buckets()
        Ac.device_arrays()
        ms, graph = timed_graph(lambda: _countsketch_csr_device(op, Ac), reps)
        byts = W.algorithmic_bytes(c, nnz)
        out.update(nnz=nnz, kernel="countsketch_csr", kernel_ms=round(ms, 4), graph_timed=graph,
                   gbs=round(byts / ms / 1e6, 1), frac_hbm=round(byts / ms / 1e6 / PEAK_HBM, 4))
        SA = _countsketch_csr_device(op, Ac)
        Sb, _ = _countsketch_dense_device(op, b.reshape(-1, 1), c.m, 1)
        # S b: one long column -> the ordered bucket walk (bitwise csr_matvec)
        vms, _ = timed_graph(lambda: _countsketch_dense_device(op, b.reshape(-1, 1), c.m, 1), reps)
        out.update(sb_ordered_walk_ms=round(vms, 4),
                   sb_gbs=round(8 * c.m / vms / 1e6, 1))
        out["qr_ms"] = round(timed(lambda: reduced_solve_device(SA, c.d, Sb[:, 0], c.d, c.n), 3), 3)
        out["qr_path"] = "cholqr2+csne" if cholqr_enabled(c.d, c.n) else "householder"
        out["householder_qr_ms"] = round(timed(lambda: qr_solve_device(SA, c.d, Sb[:, 0], c.d, c.n), 3), 3)
        out["solve"] = solve_rate(Ac, b, "countsketch", c.d, c.n)
        return out
    lda = int(A.stride(1))
    kinds = [c.kind] + (["countsketch"] if cfg_id == 5 else [])
    for kind in kinds:
        op = E.build_sketch(E.SketchSpec(kind, c.d, seed=1), c.m)
        rec = {}
        if kind == "countsketch":
            op.device_plan()
            ms, graph = timed_graph(lambda: _countsketch_dense_device(op, A, lda, c.n, b=b), reps)
            byts = W.algorithmic_bytes(c)
            rec.update(kernel_ms=round(ms, 4), graph_timed=graph, gbs=round(byts / ms / 1e6, 1),
                       frac_hbm=round(byts / ms / 1e6 / PEAK_HBM, 4))
        elif kind == "srht":
            op.device_srht()
            ms, graph = timed_graph(lambda: _srht_device(op, A, lda, c.n), reps)
            byts = 8 * c.m * c.n
            rec.update(kernel_ms=round(ms, 4), graph_timed=graph, gbs=round(byts / ms / 1e6, 1),
                       frac_hbm=round(byts / ms / 1e6 / PEAK_HBM, 4), note="A only (the SAA solve sketches [A | b] in one pass, skl_srht_dense_ab)")
        elif kind == "gaussian":
            t0 = time.perf_counter()
            G, ldg = op.device_gaussian()
            torch.cuda.synchronize()
            rec["generate_G_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
            ms = timed(lambda: _gaussian_device(op, A, lda, c.n), max(3, reps // 2))
            flops = 2.0 * c.d * c.m * c.n
            Gv = G[:, : c.m]
            cub = timed(lambda: torch.matmul(Gv, A), max(3, reps // 2))
            rec.update(kernel_ms=round(ms, 4), tflops=round(flops / ms / 1e9, 2),
                       cublas_dgemm_ms=round(cub, 4), cublas_tflops=round(flops / cub / 1e9, 2),
                       frac_of_cublas=round(cub / ms, 4))
            del Gv
        rec["solve"] = solve_rate(E.DenseMatrix(A), b, kind, c.d, c.n)
        out[kind] = rec
        del op
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    for cid in [int(x) for x in args.configs.split(",")]:
        try:
            print(json.dumps(run(cid, args.reps)), flush=True)
        except Exception as exc:  # keep going with the other configs
            print(json.dumps({"config": cid, "error": repr(exc)}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
