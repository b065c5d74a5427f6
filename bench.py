#!/usr/bin/env python
"""Benchmark of the B200 sketch engine on BASELINE.json's headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 2] [--kind countsketch]

Workload (N=1): BASELINE config 2 -- dense fp64 A of 2^20 x 256
(U diag(logspace(0,-8)) V^T, kappa = 1e8), b = A x + 1e-6 noise,
CountSketch d = 2048.  A "step" is one pass of the hot path over one batch:
S [A | b] by the CountSketch kernel (plus, for N > 1, the NCCL reduce of
the d x (n+1) partials).  value = bytes of A and b sketched per second,
whole job (weak scaling: every rank owns a 2^20-row block of an N*2^20-row
problem).  Inputs are device-resident (2 GiB/step > 126 MB L2, so no L2
flush is needed).  Reported beside it:

* roofline  -- the CountSketch kernel's algorithmic bytes / CUDA-event time
               against the measured HBM copy bandwidth (MEASURED_PEAKS.json);
* e2e       -- the same metric through the C-ABI host-buffer entry point
               (skl_countsketch_dense_host: pinned host A/b in, host SA/Sb
               out, H2D/D2H inside the timed call);
* solves    -- full SAA solves/sec through the public API on device data
               (operator build + sketch + QR + back-solve + residual), with
               the QR time reported separately;
* cpu_baseline -- the reference's algorithm (oracle port: scipy CSR @ A,
               as sketch.py:209-212 does) timed on this host on a bounded
               sample of the same workload.

``--impl reference`` prints the reference arm: the same metric measured on
the oracle port on the host cores (rank 0 only under torchrun).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profiled_traffic(kernel_regex: str):
    """DRAM bytes per launch of the timed kernel from the committed ncu
    --set full capture summaries (profiles/*countsketch*_full.json): only a
    capture whose kernel name matches the kernel this run timed counts (the
    newest such file); None otherwise."""
    import re

    best = None
    for f in sorted((ROOT / "profiles").glob("*countsketch*full*.json")):
        try:
            summ = json.loads(f.read_text())
        except Exception:
            continue
        name = str(summ.get("metrics", {}).get("Kernel Name", ""))
        if re.search(kernel_regex, name):
            best = (summ.get("dram_bytes_per_launch"), f.name, name)
    return best


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML is polled from a thread every ~1 ms (nvidia-smi's fastest loop is
    far slower than a short timed region); samples are kept only between
    __enter__ and __exit__ (none when NVML is unavailable)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4, "hw_power_brake": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, sm_max_mhz, reasons bitmask)
        self.stop_ev = threading.Event()
        self.th = None
        self.source = "nvml"

    def _poll(self):
        import pynvml

        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        self.ready.set()
        while True:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(smax), int(rs)))
            except Exception:
                pass
            if self.stop_ev.wait(0.001):
                break

    def __enter__(self):
        self.ready = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            self.ready.wait(2.0)
        except Exception:
            self.th = None
            self.source = "unavailable"
        return self

    def __exit__(self, *exc):
        self.stop_ev.set()
        if self.th is not None:
            self.th.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": self.source}
        reasons = sorted(name for name, bit in self.REASONS.items()
                         if any(r & bit for _, _, r in self.samples))
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml (1 ms poll)"}


# ----------------------------------------------------------------- CPU arms
def metric_name(cfg) -> str:
    return (f"S·A sketch GB/s (config {cfg.cfg}: CountSketch d={cfg.d}, "
            f"dense {cfg.m}x{cfg.n} fp64 per GPU)")


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_sample(cfg, A_host: np.ndarray, b_host: np.ndarray, rows, signs, reps: int,
                         threads: int | None = None):
    """Time the reference's algorithm (oracle port) on a row sample:
    `sparse_map @ A` and `sparse_map @ b` exactly as sketch.py:209-212 do,
    on A stored column-major as the reference's DenseMatrix keeps it
    (linalg.py:38).  scipy's product is single-threaded, so the sample is cut
    into `threads` row blocks whose products run concurrently (scipy drops
    the GIL inside csr_matvecs) and the d x n partials are summed -- the
    reference's own code path using every host core.
    Returns (GB/s, seconds per rep, per-rep times, threads)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    threads = threads or host_threads()
    ms = A_host.shape[0]
    cuts = np.linspace(0, ms, threads + 1).astype(np.int64)
    maps = [O.countsketch_map(rows[a:c].astype(np.int64), signs[a:c].astype(np.float64), cfg.d,
                              int(c - a)) for a, c in zip(cuts[:-1], cuts[1:])]

    def block(k):
        a, c = cuts[k], cuts[k + 1]
        return maps[k] @ A_host[a:c], maps[k] @ b_host[a:c]

    bytes_ = 8 * A_host.size + 8 * b_host.size
    times = []
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(block, range(threads)))  # warm the code path and the pool
        for _ in range(reps):
            t0 = time.perf_counter()
            parts = list(ex.map(block, range(threads)))
            SA = parts[0][0].copy()
            Sb = parts[0][1].copy()
            for pa, pb in parts[1:]:
                SA += pa
                Sb += pb
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return bytes_ / t / 1e9, t, times, threads


def cpu_stock_apply(A_host: np.ndarray, b_host: np.ndarray, rows, signs, d: int):
    """The reference's own apply as it stands (sketch.py:209-212 on the
    column-major DenseMatrix, linalg.py:38): `sparse_map @ A.data` -- scipy's
    single-threaded csr_matvecs after its internal F->C copy of A -- plus
    `sparse_map @ b`, once, on the full block."""
    from oracle import oracle as O

    smap = O.countsketch_map(np.asarray(rows, np.int64), np.asarray(signs, np.float64), d,
                             A_host.shape[0])
    t0 = time.perf_counter()
    smap @ A_host
    smap @ b_host
    t = time.perf_counter() - t0
    return {"value": round((8 * A_host.size + 8 * b_host.size) / t / 1e9, 4), "unit": "GB/s",
            "cores": 1, "seconds": round(t, 3),
            "what": "sparse_map @ A (F-ordered, incl. scipy's F->C copy) + sparse_map @ b, once"}


def cpu_reference_solve(A_host: np.ndarray, b_host: np.ndarray, d_factor: float):
    """One solve(problem, "saa", SketchSpec("countsketch", 1, SEED),
    SolverOptions(d_factor)) of the reference's algorithm on the host (the
    oracle restatement of solvers.py:296-320: operator draws, sparse_map @ A,
    numpy QR, triangular solve, ||Ax - b||), timed like the reference's
    wall_time_s (solvers.py:374/397)."""
    from oracle import oracle as O
    from paper_2409_14309_b200 import workloads as W

    t0 = time.perf_counter()
    res = O.saa_solve(A_host, b_host, "countsketch", W.SEED, d_factor)
    t = time.perf_counter() - t0
    return {"solves_per_sec": round(1.0 / t, 4), "seconds": round(t, 3),
            "residual": res["residual"], "cores": host_threads(),
            "what": "oracle saa_solve on the full block: draws + scipy csr @ A (1 thread) + "
                    "numpy QR / solve_triangular / residual (OpenBLAS, all cores)"}


def run_reference_arm(args, cfg):
    import torch

    from paper_2409_14309_b200 import workloads as W
    from paper_2409_14309_b200.rng import derive_seed

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the full config-2 block: one step = S[A|b] over all 2^20 rows
    ms = cfg.m
    c = W.config(cfg.cfg, m=ms)
    if torch.cuda.is_available():
        A, b, _ = W.make_problem(c, backend="torch")
        A_host = np.asfortranarray(A.cpu().numpy())
        b_host = b.cpu().numpy()
    else:
        A_host, b_host, _ = W.make_problem(c)
    from oracle import oracle as O

    key = O.derive_seed(derive_seed(W.SEED, "saa"), "countsketch", cfg.m)
    rows, signs = O.countsketch_draws(key, cfg.m, cfg.d)
    _, _, _, threads = cpu_reference_sample(cfg, A_host, b_host, rows, signs, args.warmup)
    _, t, times, _ = cpu_reference_sample(cfg, A_host, b_host, rows, signs, args.steps, threads)
    gbs = (8 * A_host.size + 8 * b_host.size) / t / 1e9
    sample = (f"all {ms} rows of config {cfg.cfg} (A {ms}x{cfg.n} column-major + b), "
              f"scipy CSR @ A as sketch.py:209-212, {threads} row blocks on {threads} threads; "
              f"median of {args.steps}")
    line = {
        "impl": "reference",
        "metric": metric_name(cfg),
        "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config {cfg.cfg}: dense {cfg.m}x{cfg.n} fp64 (kappa=1e8) per GPU, "
                               f"CountSketch d={cfg.d}, one pass S[A|b]",
                   "m_per_gpu": cfg.m, "n": cfg.n, "d": cfg.d, "m_sample": ms,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def launch_check(args):
    """Form the world, all-reduce (rank + 1) once, rank 0 prints what it saw."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_nccl = torch.cuda.is_available() and torch.cuda.device_count() >= world
    if use_nccl:
        torch.cuda.set_device(local)
    backend = "nccl" if use_nccl else "gloo"
    if world > 1:
        dist.init_process_group(backend)
    t = torch.tensor([rank + 1.0], dtype=torch.float64, device="cuda" if use_nccl else "cpu")
    if world > 1:
        dist.all_reduce(t)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": args.gpus, "world": world,
                          "backend": backend if world > 1 else "none",
                          "rank_sum": float(t.item()),
                          "launcher": "torchrun" if "TORCHELASTIC_RUN_ID" in os.environ
                          or "LOCAL_WORLD_SIZE" in os.environ else "none"}), flush=True)


# ----------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the check of the timed output against the oracle")
    ap.add_argument("--launch-check", action="store_true",
                    help="form the N-rank world (relaunching under torchrun if needed), "
                         "all-reduce once, print the world rank 0 saw, exit")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2409_14309_b200.launch import LaunchError, ensure_world

    if args.impl == "b200" or args.launch_check:
        # one process per GPU: without a launcher, --gpus N > 1 re-executes
        # this script under torch.distributed.run; under one, WORLD_SIZE must
        # be N -- never a silent 1-GPU run labelled N
        try:
            ensure_world(args.gpus, str(Path(__file__).resolve()), sys.argv[1:],
                         need_gpus=not args.launch_check)
        except LaunchError as exc:
            print(f"bench.py: {exc}", file=sys.stderr)
            sys.exit(2)
    if args.launch_check:
        launch_check(args)
        return

    from paper_2409_14309_b200 import workloads as W

    cfg = W.config(args.config)
    if cfg.kind != "countsketch" or cfg.gen == "csr":
        cfg = W.config(args.config, kind="countsketch")
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2409_14309_b200 as E
    from paper_2409_14309_b200 import _native
    from paper_2409_14309_b200.distributed import ShardPlan, local_partial_device, shard_rows
    from paper_2409_14309_b200.rng import derive_seed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # SKL_BENCH_PEER=1 runs the fused peer-slot reduce even at N = 1 (a
    # one-rank group), so the N > 1 code path can be exercised on one GPU
    force_peer = bool(os.environ.get("SKL_BENCH_PEER"))
    grouped = world > 1 or force_peer
    if grouped:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    # ---- data: every rank owns a full config-sized row block (weak scaling)
    m_loc, n, d = cfg.m, cfg.n, cfg.d
    m_total = m_loc * world
    A, b, _ = W.make_problem(W.config(cfg.cfg, m=m_loc), seed=W.SEED + rank, backend="torch")
    lda = int(A.stride(1))
    spec = E.SketchSpec("countsketch", d, seed=derive_seed(W.SEED, "saa"))
    r0, r1 = shard_rows(m_total, world, rank)
    assert r1 - r0 == m_loc

    def build_operator():
        E.clear_operator_cache()
        o = E.build_sketch(spec, m_total)
        pl = ShardPlan(o, r0, r1)
        pl.device_plan()
        torch.cuda.synchronize()
        return o, pl

    build_operator()  # first call loads kernels
    builds = []
    for _ in range(3):
        t_build0 = time.perf_counter()
        op, plan = build_operator()
        builds.append(time.perf_counter() - t_build0)
    build_s = statistics.median(builds)

    stream = torch.cuda.current_stream()
    ld = (d + 1) // 2 * 2
    # column-major d x (n+1) view of a contiguous buffer: the collective
    # reduces the buffer itself (NCCL needs contiguous tensors)
    outbuf = torch.empty((n + 1, ld), dtype=torch.float64, device="cuda")
    out = outbuf.t()[:d]
    cs_plan = plan.device_plan()
    # N > 1: every rank's kernel writes its partial into its own symmetric
    # buffer; the ranks then reduce-scatter the partials over NVLink in rank
    # order straight into rank 0's result (distributed.PeerReduce); one NCCL
    # reduce where symmetric memory is unavailable.
    from paper_2409_14309_b200.distributed import peer_reduce_or_none

    peer = peer_reduce_or_none(d, n + 1) if grouped else None
    collective = ("peer-reduce-scatter (symmetric memory, skl_reduce_peers)" if peer is not None
                  else ("nccl-reduce" if world > 1 else "none"))
    # one line per rank on stderr: the world this run actually formed
    print(f"[bench] rank {rank}/{world} local {local} device {torch.cuda.current_device()} "
          f"({torch.cuda.get_device_name()}) collective={collective}", file=sys.stderr, flush=True)

    def apply():
        if peer is not None:
            base = peer.partial_ptr()
            cs_plan.apply(A, m_loc, n, lda, b, base, peer.ld, base + 8 * peer.ld * n,
                          partitions=1, stream=stream.cuda_stream)
        else:
            cs_plan.apply(A, m_loc, n, lda, b, out, ld, out[:, n], partitions=1,
                          stream=stream.cuda_stream)

    def collect():
        if peer is not None:
            peer.finish(out, ld)
        elif world > 1:
            dist.reduce(outbuf, dst=0)

    def step():
        apply()
        collect()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            k_ev[i][0].record(stream)
            apply()
            k_ev[i][1].record(stream)
            collect()
        stop.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    total_ms = start.elapsed_time(stop)
    kern_ms = [a.elapsed_time(bb) for a, bb in k_ev]
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    bytes_local = W.algorithmic_bytes(W.config(cfg.cfg, m=m_loc))
    value = bytes_local * world / (ms_per_step * 1e-3) / 1e9
    kern_avg = statistics.mean(kern_ms)
    achieved = bytes_local / (kern_avg * 1e-3) / 1e9
    peak, peak_src = hbm_peak()

    # ---- full SAA solves through the public API (device data), QR separately
    solve = None
    if not args.no_solve and world == 1:
        prob = E.LeastSquaresProblem(A=E.DenseMatrix(A), b=E.Vector(b))
        sspec = E.SketchSpec("countsketch", 1, seed=W.SEED)
        opts = E.SolverOptions(d_factor=d / n)
        E.solve(prob, "saa", sspec, opts)  # warm (kernels, pools)
        reps = 5
        cold = []
        for _ in range(3):  # operator rebuilt every solve, as the reference does
            E.clear_operator_cache()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            E.solve(prob, "saa", sspec, opts)
            torch.cuda.synchronize()
            cold.append(time.perf_counter() - t0)
        E.solve(prob, "saa", sspec, opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            res = E.solve(prob, "saa", sspec, opts)
        torch.cuda.synchronize()
        solve_s = (time.perf_counter() - t0) / reps
        cold_s = statistics.median(cold)
        # the reduced solve alone on the sketched matrix, through the path
        # solve() takes (CholeskyQR2 + refinement when eligible), and the
        # Householder factorisation it falls back to, for comparison
        from paper_2409_14309_b200.linalg import (cholqr_enabled, qr_solve_device,
                                                  qr_solve_device_async)

        SAb = out

        def reduced_ms(fn):
            qa, qb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fn()
            torch.cuda.synchronize()
            qa.record(stream)
            for _ in range(reps):
                fn()
            qb.record(stream)
            torch.cuda.synchronize()
            return qa.elapsed_time(qb) / reps

        qr_ms = reduced_ms(lambda: qr_solve_device_async(SAb[:, :n], ld, SAb[:, n], d, n))
        hh_ms = reduced_ms(lambda: qr_solve_device(SAb[:, :n], ld, SAb[:, n], d, n))
        qr_path = "cholqr2+csne" if cholqr_enabled(d, n) else "householder"
        # host-input solves: pinned host carriers through solve(); the sketch
        # streams row blocks of A to the device under the kernel and keeps the
        # device copy for the residual pass (skl_countsketch_dense_owned_host
        # with A_dev_keep), x comes back to the host
        from paper_2409_14309_b200._device import pinned_empty_f64

        Ah_solve = pinned_empty_f64((m_loc, n), fortran=True)
        Ah_solve[...] = A.cpu().numpy()
        bh_solve = pinned_empty_f64((m_loc,))
        bh_solve[...] = b.cpu().numpy()
        prob_h = E.LeastSquaresProblem(A=E.DenseMatrix(Ah_solve), b=E.Vector(bh_solve))
        res_h = E.solve(prob_h, "saa", sspec, opts)
        t0 = time.perf_counter()
        for _ in range(3):
            res_h = E.solve(prob_h, "saa", sspec, opts)
        host_s = (time.perf_counter() - t0) / 3
        host_x_err = float(np.linalg.norm(res_h.x.data - res.x.data.cpu().numpy())
                           / np.linalg.norm(res_h.x.data))
        # batched solves: solve_many() enqueues independent solves on two
        # streams with one host synchronisation, so one problem's reduced
        # solve runs beside the next one's HBM passes (every solve still
        # fully recomputed: 16 sketches, 16 reduced solves, 16 residuals)
        batch = [prob] * 16
        E.solve_many(batch, "saa", sspec, opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(2):
            many = E.solve_many(batch, "saa", sspec, opts)
        torch.cuda.synchronize()
        batch_s = (time.perf_counter() - t0) / (2 * len(batch))
        assert all(r.residual_norm == res.residual_norm for r in many)
        # sketch-and-precondition: LSQR preconditioned by R
        sap_opts = E.SolverOptions(d_factor=d / n)
        E.solve(prob, "sap", sspec, sap_opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            sap = E.solve(prob, "sap", sspec, sap_opts)
        torch.cuda.synchronize()
        sap_s = (time.perf_counter() - t0) / 3
        solve = {"solves_per_sec": round(1.0 / solve_s, 3), "ms_per_solve": round(solve_s * 1e3, 3),
                 "sap_solves_per_sec": round(1.0 / sap_s, 3), "sap_ms_per_solve": round(sap_s * 1e3, 2),
                 "sap_iterations": sap.iterations, "sap_residual": sap.residual_norm,
                 "solves_per_sec_cold": round(1.0 / cold_s, 3),
                 "batched_solves_per_sec": round(1.0 / batch_s, 3),
                 "batched_ms_per_solve": round(batch_s * 1e3, 3),
                 "ms_per_solve_cold": round(cold_s * 1e3, 3),
                 "qr_solve_ms": round(qr_ms, 3), "qr_path": qr_path,
                 "householder_qr_solve_ms": round(hh_ms, 3), "residual": res.residual_norm,
                 "host_solves_per_sec": round(1.0 / host_s, 3),
                 "host_ms_per_solve": round(host_s * 1e3, 3),
                 "host_vs_device_x_rel_diff": host_x_err,
                 "operator_build_ms": round(build_s * 1e3, 2),
                 "includes": "sketch S[A|b], QR, back-solve, residual on device-resident A; "
                             "the *_cold figures also rebuild the operator (device RNG + "
                             "device plan) every solve, as the reference does; host_* solves "
                             "take pinned host A,b (H2D streamed under the sketch, device copy "
                             "kept for the residual, x to the host); batched_* take 16 "
                             "independent solves through solve_many (two streams, one host "
                             "sync per batch; each solve fully recomputed)"}

    # ---- e2e through the C-ABI host-buffer entry point
    e2e = None
    if not args.no_e2e:
        from paper_2409_14309_b200._device import pinned_empty_f64

        Ah = pinned_empty_f64((m_loc, n), fortran=True)
        Ah[...] = A.cpu().numpy()
        bh = pinned_empty_f64((m_loc,))
        bh[...] = b.cpu().numpy()
        SAh = np.empty((d, n), order="F")
        Sbh = np.empty(d)

        def e2e_call():
            cs_plan.apply_host(Ah, m_loc, n, m_loc, bh, SAh, d, Sbh, stream=stream.cuda_stream)

        e2e_call()
        reps = 3
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            e2e_call()
            ts.append(time.perf_counter() - t0)
        te = statistics.median(ts)
        if world > 1:  # whole job: all ranks' bytes over the slowest rank's time
            t = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": round(bytes_local * world / te / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": bytes_local, "d2h_bytes_per_step": 8 * d * (n + 1),
               "ms_per_step": round(te * 1e3, 3),
               "path": f"{'skl_countsketch_dense_owned_host' if cs_plan.kind == 'owned' else 'skl_countsketch_dense_host'}"
                       " (pinned host A,b -> host SA,Sb)"}
        if world == 1:
            # parity of the timed output against the device run (bitwise)
            assert np.array_equal(SAh, out[:, :n].cpu().numpy())

    # parity of the timed output: the device S[A|b] of the timed loop against
    # the oracle's csr_matvecs fold (threaded C restatement), bitwise
    parity = None
    if world == 1 and not args.no_parity:
        from oracle import clib

        A_host = np.asfortranarray(A.cpu().numpy())
        b_host = b.cpu().numpy()
        rows_h, signs_h = op.rows, op.signs
        want = clib.countsketch_apply_mt(rows_h, signs_h, d, A_host)
        want_b = clib.countsketch_apply_mt(rows_h, signs_h, d, b_host)
        got = out.cpu().numpy()
        bitwise = bool(np.array_equal(got[:, :n], want) and np.array_equal(got[:, n], want_b))
        parity = {"timed_output_vs_oracle": "bitwise" if bitwise else "MISMATCH",
                  "oracle": "oracle/c/apply_oracle.c (scipy csr_matvecs fold, sketch.py:209-212)"}
        if not bitwise:
            print("bench.py: timed S[A|b] differs from the oracle", file=sys.stderr)
            sys.exit(3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU leg: rank 0 at N = 1 only
        A_host = np.asfortranarray(A.cpu().numpy()) if parity is None else A_host
        b_host = b.cpu().numpy() if parity is None else b_host
        gbs, t, _, threads = cpu_reference_sample(cfg, A_host, b_host, op.rows, op.signs, 3)
        stock = cpu_stock_apply(A_host, b_host, op.rows, op.signs, d)
        ref_solve = cpu_reference_solve(A_host, b_host, d / n)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"the full config-{cfg.cfg} block ({m_loc} x {n} column-major + b), "
                         f"scipy CSR @ A (the reference's csr_matvecs path, sketch.py:209-212) in "
                         f"{threads} row blocks on {threads} threads, median of 3 = "
                         f"{t * 1e3:.1f} ms",
               "stock_single_thread": stock,
               "reference_saa_solve": ref_solve}
    if cs_plan.kind == "owned":
        threads = 32 * cs_plan.warps
        nsl = 4 if d <= threads * 4 else 8
        kernel_name = f"skl::countsketch_owned_kernel<{threads}, 0, {nsl}>"
        kernel_rx = rf"countsketch_owned_kernel<{threads},\s*(0|false),\s*{nsl}>"
    else:
        kernel_name = f"skl::countsketch_dense_kernel<{32 * cs_plan.warps}, ...>"
        kernel_rx = rf"countsketch_dense_kernel<{32 * cs_plan.warps}\b"
    traffic = profiled_traffic(kernel_rx)
    if rank == 0:
        line = {
            "metric": metric_name(cfg),
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config {cfg.cfg}: dense {m_loc}x{n} fp64 (kappa=1e8) per GPU, "
                                   f"CountSketch d={d}, one pass S[A|b]"
                                   + (" + reduce of the d x (n+1) partials" if world > 1 else ""),
                       "collective": collective,
                       "ranks": world,
                       "launcher": ("torchrun" if "LOCAL_WORLD_SIZE" in os.environ
                                    else "none (single process)"),
                       "m_per_gpu": m_loc, "n": n, "d": d, "m_total": m_total,
                       "parallelism": f"rows sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2 (2 GiB of A per GPU per step); no flush"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic[0] if traffic else None,
                         "traffic_source": (f"profiles/{traffic[1]}: {traffic[2]}" if traffic
                                            else "no ncu capture of this kernel"),
                         "peak_source": peak_src,
                         "kernel": kernel_name,
                         "kernel_ms": round(kern_avg, 4),
                         "algorithmic_bytes_per_launch": bytes_local,
                         "frac_of_8TBps": round(achieved / 8000.0, 4)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "parity": parity,
            "clocks": clocks.summary(),
            # our kernels per timed step: the sketch, plus this rank's block of
            # the peer reduce
            "gpu_launches": args.steps * (2 if peer is not None else 1),
        }
        if solve:
            line["solve"] = solve
        print(json.dumps(line), flush=True)
    if grouped:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
