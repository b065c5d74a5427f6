"""Row-sharded sketch-and-apply across GPUs.

Row block k of A (and b) lives on rank k.  Every rank sketches its block
with the hashes of its *global* row indices -- the operator is realised
once for the global m, exactly as the reference would build it
(sketch.py:93-103) -- producing a partial d x (n+1) [SA | Sb].  One
NCCL reduce (sum, fp64) to rank 0 completes S[A | b]; rank 0 solves the
reduced problem, broadcasts x, and the residual norm is an all-reduce of
the per-block squared residuals.

The sum over ranks changes the floating-point order relative to the
single-pass fold, so the result is within ~1e-15 relative of the 1-GPU
(bitwise-reference) sketch, not bitwise.  Process layout: one process per
GPU, launched by torchrun; ``torch.distributed`` (backend "nccl") is only
plumbing for the reduce/broadcast.
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np

from . import _native
from ._device import current_stream, device_f64, require_cuda, to_device, torch
from .sketch import SHARD_ALIGN, CountSketchPlan, SketchOperator, build_sketch


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [r0, r1) of rank ``rank``; blocks start on
    multiples of SHARD_ALIGN rows (keeps row blocks of a shared array
    16-byte aligned and the shards near-equal)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    chunks = math.ceil(m / SHARD_ALIGN)
    c0 = chunks * rank // world
    c1 = chunks * (rank + 1) // world
    return min(m, c0 * SHARD_ALIGN), min(m, c1 * SHARD_ALIGN)


class ShardPlan:
    """The part of a global CountSketch operator that rank ``rank`` needs:
    hashes of global rows [r0, r1) and their device plan."""

    def __init__(self, op: SketchOperator, r0: int, r1: int):
        if op.kind != "countsketch":
            raise ValueError("row sharding is implemented for CountSketch operators")
        self.op, self.r0, self.r1 = op, r0, r1
        self.d = op.target_dim
        self.rows = np.ascontiguousarray(op.rows[r0:r1])
        self.signs = np.ascontiguousarray(op.signs[r0:r1])
        self._plan = None

    def device_plan(self) -> CountSketchPlan:
        if self._plan is None:
            self._plan = CountSketchPlan(self.rows, self.signs, self.d)
        return self._plan


def local_partial_device(plan: ShardPlan, A_local, lda: int, b_local):
    """Partial [SA | Sb] of one row block on this rank's GPU: a d x (n+1)
    column-major tensor whose last column is the partial Sb."""
    require_cuda()
    m_loc = plan.r1 - plan.r0
    n = A_local.shape[1]
    d = plan.d
    ld = (d + 1) // 2 * 2  # keeps the Sb column 16-byte aligned
    out = device_f64((d, n + 1), fortran=True, ld=ld)
    plan.device_plan().apply(A_local, m_loc, n, lda, b_local, out, ld, out[:, n], partitions=1)
    return out


def reduce_partials(partial, dist, group=None, dst: int = 0):
    """Sum the per-rank partials onto rank ``dst`` (one NCCL reduce)."""
    dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partial


def sharded_sketch_and_apply(A_local, b_local, m_total: int, spec, dist, group=None,
                             local_apply: Callable | None = None, solve_reduced=None,
                             residual_local=None):
    """SAA over row-sharded data.  Returns (x, residual_norm, d) on every rank.

    ``local_apply(plan, A_local, b_local) -> partial`` defaults to the CUDA
    kernel; ``solve_reduced(partial) -> x`` and ``residual_local(A, b, x)``
    default to the device QR / residual kernels.  The hooks exist so the
    host-side sharding and collective logic can be exercised on CPU (gloo).
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    r0, r1 = shard_rows(m_total, world, rank)
    if A_local.shape[0] != r1 - r0:
        raise ValueError(f"rank {rank} holds {A_local.shape[0]} rows, expected {r1 - r0}")
    op = build_sketch(spec, m_total)
    plan = ShardPlan(op, r0, r1)
    n = A_local.shape[1]
    if local_apply is None:
        lda = int(A_local.stride(1)) if n > 1 else A_local.shape[0]
        partial = local_partial_device(plan, A_local, lda, b_local)
    else:
        partial = local_apply(plan, A_local, b_local)
    reduce_partials(partial, dist, group)
    d = plan.d
    if rank == 0:
        if solve_reduced is None:
            from .linalg import qr_solve_device

            x, _, _ = qr_solve_device(partial[:, :n], int(partial.stride(1)), partial[:, n], d, n)
        else:
            x = solve_reduced(partial)
    else:
        x = torch.empty(n, dtype=torch.float64, device=partial.device)
    dist.broadcast(x, src=0, group=group)
    if residual_local is None:
        out = np.zeros(1)
        lda = int(A_local.stride(1)) if n > 1 else A_local.shape[0]
        _native.call("skl_residual_dense", _native.ptr(A_local), A_local.shape[0], n, lda,
                     _native.ptr(x), _native.ptr(b_local), _native.ptr(out), current_stream())
        r2 = torch.tensor([out[0] ** 2], dtype=torch.float64, device=partial.device)
    else:
        r2 = residual_local(A_local, b_local, x)
    dist.all_reduce(r2, op=dist.ReduceOp.SUM, group=group)
    return x, float(torch.sqrt(r2).item()), d
