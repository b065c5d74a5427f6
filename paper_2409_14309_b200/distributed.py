"""Row-sharded sketch-and-apply across GPUs.

Row block k of A (and b) lives on rank k.  Every rank sketches its block
with the operator realised once for the GLOBAL m, exactly as the reference
would build it (sketch.py:84-127) -- CountSketch hashes of global rows,
SRHT sign/sample with the shard's block offset, the Gaussian column block --
producing a partial d x (n+1) [SA | Sb].  One
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
    """The part of a global operator that the rank owning rows [r0, r1) needs.

    * countsketch: the hashes/signs of the global rows [r0, r1) and their
      device plan (the hash of row j is the reference's draw for GLOBAL j);
    * srht: the packed sign words of the shard's 4096-row blocks (a slice of
      the global packing, shards are block aligned) plus the global sample;
      the kernel adds the (-1)^popc(p_hi & j_hi) factor for the shard's
      block offset, i.e. H_m = H_G (x) H_{m/G} over (shard, local) bits;
    * gaussian: the column block S[:, r0:r1] of the row-major d x m matrix
      (the full G is generated on each rank -- the ziggurat stream is
      sequential -- and the GEMM reads only the block)."""

    def __init__(self, op: SketchOperator, r0: int, r1: int):
        if op.kind not in ("countsketch", "srht", "gaussian"):
            raise ValueError(f"row sharding is not implemented for {op.kind!r} operators")
        if op.kind == "srht":
            B = min(op.padded_dim, 4096)
            if r0 % B:
                raise ValueError(f"SRHT shard start {r0} is not a multiple of the block {B}")
        self.op, self.r0, self.r1 = op, r0, r1
        self.kind = op.kind
        self.d = op.target_dim
        self._plan = None

    @property
    def rows(self):
        return np.ascontiguousarray(self.op.rows[self.r0:self.r1])

    @property
    def signs(self):
        return np.ascontiguousarray(self.op.signs[self.r0:self.r1])

    def device_plan(self) -> CountSketchPlan:
        if self._plan is None:
            h = self.op._cache().get("hash") if torch.cuda.is_available() else None
            if h is not None and _native.plan_geometry(self.d)[0] == "owned":
                # slices of the device draws: the plan is built on the device
                self._plan = CountSketchPlan.from_device(h[0][self.r0:self.r1],
                                                         h[1][self.r0:self.r1], self.d,
                                                         self.r1 - self.r0)
            else:
                self._plan = CountSketchPlan(self.rows, self.signs, self.d)
        return self._plan

    def device_srht_words(self):
        """Packed sign words of this shard's blocks (device view)."""
        signs, _ = self.op.device_srht()
        B = min(self.op.padded_dim, 4096)
        per_block = int(_native.lib().skl_srht_sign_words(B))
        return signs[(self.r0 // B) * per_block:]


def local_partial_device(plan: ShardPlan, A_local, lda: int, b_local):
    """Partial [SA | Sb] of one row block on this rank's GPU: a d x (n+1)
    column-major tensor whose last column is the partial Sb."""
    require_cuda()
    m_loc = plan.r1 - plan.r0
    n = A_local.shape[1]
    d = plan.d
    ld = (d + 1) // 2 * 2  # keeps the Sb column 16-byte aligned
    out = device_f64((d, n + 1), fortran=True, ld=ld)
    st = current_stream()
    if plan.kind == "countsketch":
        plan.device_plan().apply(A_local, m_loc, n, lda, b_local, out, ld, out[:, n],
                                 partitions=1)
    elif plan.kind == "srht":
        words = plan.device_srht_words()
        _, sample = plan.op.device_srht()
        for src, ncol, ldsrc, dst in ((A_local, n, lda, out), (b_local, 1, m_loc, out[:, n])):
            _native.call("skl_srht_dense_shard", _native.ptr(src), m_loc, ncol, ldsrc,
                         _native.ptr(words), _native.ptr(sample), plan.op.padded_dim, d, plan.r0,
                         _native.ptr(dst), ld, st)
    else:
        G, ldg = plan.op.device_gaussian()
        Gs = G[:, plan.r0:]
        for src, ncol, ldsrc, dst in ((A_local, n, lda, out), (b_local, 1, m_loc, out[:, n])):
            _native.call("skl_gemm_f64", _native.ptr(Gs), ldg, _native.ptr(src), ldsrc,
                         _native.ptr(dst), ld, d, ncol, m_loc, 0, st)
    return out


def reduce_partials(partial, dist, group=None, dst: int = 0):
    """Sum the per-rank partials onto rank ``dst`` (one NCCL reduce).  The
    d x (n+1) column-major partial is reduced through its contiguous
    transpose (collectives need contiguous buffers)."""
    flat = partial.t()
    if flat.is_contiguous():
        dist.reduce(flat, dst=dst, op=dist.ReduceOp.SUM, group=group)
    else:
        tmp = flat.contiguous()
        dist.reduce(tmp, dst=dst, op=dist.ReduceOp.SUM, group=group)
        flat.copy_(tmp)
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
