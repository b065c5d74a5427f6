"""Single-process multi-device sketch-and-apply: ``solve(..., opts)`` with
``SolverOptions(devices=(0, 1, ...))``.

SURVEY.md §5 asks for a multi-GPU path that needs no launcher, so the
Python ``solve()`` API (/root/reference/pkg/src/sketchls/solvers.py:364-398)
can use every GPU of the box.  One host thread drives all devices, each
through its own stream: row block k of A and b goes to ``devices[k]``
(host carriers are uploaded block by block; device carriers are copied peer
to peer), every device sketches its block with the global operator's shard
plan (distributed.ShardPlan: the hashes of the global rows, the SRHT block
offset, the Gaussian column block -- generated in bands, each device parsing
~1/N of the operator's ziggurat stream, then exchanged; see
gaussian_column_blocks), the partial d x (n+1) sketches are
copied to ``devices[0]`` and summed there in device order
(skl_reduce_peers: the same fixed-order fold as the multi-process path),
the reduced QR solve runs on ``devices[0]``, and every device computes its
block's squared residual against x.

Row blocks are multiples of 8192 rows (SHARD_ALIGN), so an A with fewer
than 8192 x len(devices) rows runs on the first devices only.  A device may
appear more than once (``devices=(0, 0, 0, 0)``): the blocks
are then processed as separate shards on that device -- the shard/reduce
logic of an N-GPU run, exercised on one GPU (the tests do this).  Results
are within ~1e-15 of the one-device sketch (the per-shard partial sums
change the fp64 association), not bitwise.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from ._device import current_stream, require_cuda, to_device, torch
from .distributed import CsrBlock, ShardPlan, csr_row_block, local_partial_device, partial_ld
from .distributed import band_bounds, band_pieces, residual_sq_local, shard_rows
from .errors import SpecError
from .linalg import DenseMatrix, SparseMatrix
from .sketch import SHARD_ALIGN

MAX_DEVICES = 16
SHARDED_KINDS = ("countsketch", "srht", "gaussian")


def check_devices(devices) -> tuple[int, ...]:
    """Validate a device list (SolverOptions.devices)."""
    devs = tuple(int(d) for d in devices)
    if not devs:
        raise SpecError("devices must be a nonempty sequence of CUDA device indices")
    if len(devs) > MAX_DEVICES:
        raise SpecError(f"at most {MAX_DEVICES} devices are supported, got {len(devs)}")
    if any(d < 0 for d in devs):
        raise SpecError(f"device indices must be >= 0, got {devs}")
    if torch is not None and torch.cuda.is_available():
        have = torch.cuda.device_count()
        if any(d >= have for d in devs):
            raise SpecError(f"devices {devs} out of range: this node has {have} CUDA device(s)")
    return devs


def _dense_block(A: DenseMatrix, r0: int, r1: int, dev: int):
    """Rows [r0, r1) of a dense carrier on device ``dev`` (column-major)."""
    n = A.cols
    m_loc = r1 - r0
    if not A.on_device:
        with torch.cuda.device(dev):
            return to_device(np.asfortranarray(A.data[r0:r1])), m_loc
    src = A.data[r0:r1]
    if src.device.index == dev:
        return src, A.ld  # a view: same leading dimension
    ld = (m_loc + 1) // 2 * 2
    out = torch.empty_strided((m_loc, n), (1, ld), dtype=torch.float64,
                              device=torch.device("cuda", dev))
    out.copy_(src)
    return out, ld


def _vec_block(b, r0: int, r1: int, dev: int):
    if isinstance(b, np.ndarray):
        with torch.cuda.device(dev):
            return to_device(np.ascontiguousarray(b[r0:r1]))
    return b[r0:r1].to(torch.device("cuda", dev)).contiguous()


def _band_begin(op, seg0: int, seg1: int):
    h = ctypes.c_void_p()
    _native.call("skl_gaussian_band_begin", op.key, seg0, seg1, ctypes.byref(h), None,
                 current_stream())
    return h


def gaussian_column_blocks(op, devs, spans):
    """The Gaussian operator's column blocks S[:, r0:r1] for row shards
    ``spans`` on devices ``devs``, generated in bands: device k parses only
    segment band k of the stream (skl_gaussian_band_*), the host prefix-sums
    the bands' normal counts, every device writes its band's normals (rows
    of S), and the bands are exchanged so device k holds the columns its
    shard multiplies.  Each device generates ~1/N of the d x m operator
    instead of all of it.  Returns [(block d x w_k, ld)], bit-identical to
    the single-device G[:, r0:r1]."""
    _native.install_gaussian_tables()
    lib = _native.lib()
    d, m = op.target_dim, op.source_dim
    N = d * m
    seg_words = int(lib.skl_gaussian_segment_words())
    world = len(devs)
    bounds = band_bounds(N, world, seg_words)
    handles, counts = [None] * world, [0] * world
    for k, dev in enumerate(devs):  # enqueue every band before waiting on any
        with torch.cuda.device(dev):
            handles[k] = _band_begin(op, bounds[k], bounds[k + 1])
    for k, dev in enumerate(devs):
        with torch.cuda.device(dev):
            c = ctypes.c_int64()
            _native.call("skl_gaussian_band_count", handles[k], ctypes.byref(c), current_stream())
            counts[k] = int(c.value)
    while sum(counts) < N:  # too few words: extend the last band
        dev = devs[-1]
        with torch.cuda.device(dev):
            lib.skl_gaussian_band_free(handles[-1], ctypes.c_void_p(current_stream()))
            bounds[-1] += (bounds[-1] - bounds[-2]) // 8 + 16
            handles[-1] = _band_begin(op, bounds[-2], bounds[-1])
            c = ctypes.c_int64()
            _native.call("skl_gaussian_band_count", handles[-1], ctypes.byref(c),
                         current_stream())
            counts[-1] = int(c.value)
    firsts = [sum(counts[:k]) for k in range(world)]
    ldg = (m + 31) // 32 * 32
    div = math.sqrt(d)
    bands = []  # (tensor rows x ldg, row0, t0, t1)
    for k, dev in enumerate(devs):
        t0, t1 = min(N, firsts[k]), min(N, firsts[k] + counts[k])
        with torch.cuda.device(dev):
            if t1 <= t0:
                lib.skl_gaussian_band_free(handles[k], ctypes.c_void_p(current_stream()))
                bands.append(None)
                continue
            row0, row1 = t0 // m, (t1 - 1) // m + 1
            band = torch.empty((row1 - row0, ldg), dtype=torch.float64,
                               device=torch.device("cuda", dev))
            _native.call("skl_gaussian_band_write", handles[k], firsts[k], N, m, row0,
                         _native.ptr(band), ldg, div, current_stream())
            bands.append((band, row0, t0, t1))
    blocks = []
    for (r0, r1), dev in zip(spans, devs):
        w = r1 - r0
        ldb = (w + 31) // 32 * 32
        with torch.cuda.device(dev):
            blk = torch.empty((d, ldb), dtype=torch.float64, device=torch.device("cuda", dev))
            for bd in bands:
                if bd is None:
                    continue
                band, row0, t0, t1 = bd
                for ia, ib, a, c in band_pieces(t0, t1, m, r0, r1):
                    blk[ia:ib, a - r0:c - r0].copy_(band[ia - row0:ib - row0, a:c])
            blocks.append((blk, ldb))
    for dev in set(devs):
        torch.cuda.synchronize(dev)
    return blocks


def sketch_and_apply_devices(op, A, b, devices):
    """Row-sharded S[A | b] over ``devices`` followed by the reduced solve on
    devices[0].  Returns (x tensor on devices[0], residual norm)."""
    require_cuda()
    if op.kind not in SHARDED_KINDS:
        raise SpecError(f"multi-device sketching supports {SHARDED_KINDS}, got {op.kind!r}")
    m, n, d = A.rows, A.cols, op.target_dim
    # row blocks are SHARD_ALIGN (8192) rows: a short A uses the first devices only
    devs = check_devices(devices)[:max(1, -(-m // SHARD_ALIGN))]
    world = len(devs)
    ld = partial_ld(d)
    slot = (n + 1) * ld
    dev0 = devs[0]
    spans = [shard_rows(m, world, k) for k in range(world)]
    # shard plans (per-shard hashes, plans, bucket lists) are cached with the
    # operator, like its one-device plan
    plans = op._host.get(("shard_plans", devs))
    if plans is None:
        plans = op._host[("shard_plans", devs)] = [ShardPlan(op, r0, r1) for r0, r1 in spans]
    gblocks = None
    if op.kind == "gaussian":
        key = ("gauss_blocks", devs)
        gblocks = op._host.get(key)
        if gblocks is None:  # per-device bands of the stream, exchanged (cached)
            gblocks = op._host[key] = gaussian_column_blocks(op, devs, spans)
    caller = torch.cuda.current_stream(dev0)
    start = torch.cuda.Event()
    start.record(caller)
    shards = []
    # 1. per-device row blocks and partials, each device on its own stream
    for k, dev in enumerate(devs):
        r0, r1 = spans[k]
        with torch.cuda.device(dev):
            st = torch.cuda.Stream(dev)
            st.wait_event(start)
            with torch.cuda.stream(st):
                if isinstance(A, SparseMatrix):
                    A_loc, lda = csr_row_block(A, r0, r1, device=dev), 0
                else:
                    A_loc, lda = _dense_block(A, r0, r1, dev)
                b_loc = _vec_block(b.data, r0, r1, dev)
                plan = plans[k]
                if gblocks is not None:
                    plan.gaussian_block = gblocks[k]
                part = torch.empty(slot, dtype=torch.float64, device=torch.device("cuda", dev))
                local_partial_device(plan, A_loc, lda, b_loc, dest=part.data_ptr())
                done = torch.cuda.Event()
                done.record(st)
        shards.append((dev, st, A_loc, lda, b_loc, part, done))
    # 2. partials to devices[0] (peer copies), fixed-order sum there
    with torch.cuda.device(dev0):
        parts = []
        for dev, st, _, _, _, part, done in shards:
            caller.wait_event(done)
            if dev != dev0:
                with torch.cuda.stream(caller):
                    part = part.to(torch.device("cuda", dev0), non_blocking=True)
            part.record_stream(caller)  # allocated on the shard's stream, read on caller's
            parts.append(part)
        with torch.cuda.stream(caller):
            total = torch.empty(slot, dtype=torch.float64, device=torch.device("cuda", dev0))
            _native.call("skl_reduce_peers", _native.ptr_array([p.data_ptr() for p in parts]),
                         world, 0, slot, total.data_ptr(), current_stream())
            red = total.view(n + 1, ld).t()
            from .linalg import reduced_solve_device

            x = reduced_solve_device(red[:d, :n], ld, red[:d, n], d, n)
            x_done = torch.cuda.Event()
            x_done.record(caller)
    # 3. per-block squared residuals against x
    r2 = 0.0
    for dev, st, A_loc, lda, b_loc, _, _ in shards:
        with torch.cuda.device(dev), torch.cuda.stream(st):
            st.wait_event(x_done)
            xk = x if dev == dev0 else x.to(torch.device("cuda", dev), non_blocking=True)
            xk.record_stream(st)
            r2 += residual_sq_local(A_loc, lda, b_loc, xk)
    caller.wait_stream(shards[-1][1])
    for dev, st, *_ in shards:
        torch.cuda.current_stream(dev).wait_stream(st)
    return x, float(np.sqrt(r2))


__all__ = ["band_pieces", "check_devices", "gaussian_column_blocks", "sketch_and_apply_devices",
           "CsrBlock"]
