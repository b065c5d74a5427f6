"""Row-sharded sketch-and-apply across GPUs.

Row block k of A (and b) lives on rank k.  Every rank sketches its block
with the operator realised once for the GLOBAL m, exactly as the reference
would build it (sketch.py:84-127) -- CountSketch hashes of global rows,
SRHT sign/sample with the shard's block offset, the Gaussian column block --
producing a partial d x (n+1) [SA | Sb].

The reduce is fused with the sketch (``PeerSlots``): every rank's kernel
writes its partial straight into its own slot of rank 0's symmetric buffer
(NVLink peer stores from the kernel's epilogue, overlapping the CTAs still
streaming A), a device-side barrier orders the slots, and rank 0 sums them
in rank order (``skl_sum_slots``) -- deterministic for a given world size.
Where symmetric memory is unavailable (or on CPU with gloo, in the tests)
the partials are combined by one collective reduce instead.  Rank 0 solves
the reduced problem, broadcasts x, and the residual norm is an all-reduce
of the per-block squared residuals.

The sum over ranks changes the floating-point order relative to the
single-pass fold, so the result is within ~1e-15 relative of the 1-GPU
(bitwise-reference) sketch, not bitwise.  Process layout: one process per
GPU, launched by torchrun; ``torch.distributed`` is the plumbing (process
group, symmetric-memory rendezvous, broadcast).
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np

from . import _native
from ._device import current_stream, device_f64, require_cuda, torch
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


def partial_ld(d: int) -> int:
    """Leading dimension of a d x (n+1) partial (keeps the Sb column 16-byte
    aligned)."""
    return (d + 1) // 2 * 2


def local_partial_device(plan: ShardPlan, A_local, lda: int, b_local, dest: int | None = None):
    """Partial [SA | Sb] of one row block on this rank's GPU: a d x (n+1)
    column-major tensor (ld ``partial_ld(d)``) whose last column is the
    partial Sb.  With ``dest`` (a device address, e.g. this rank's slot in
    a peer's symmetric buffer) the kernels write there instead and None is
    returned."""
    require_cuda()
    m_loc = plan.r1 - plan.r0
    n = A_local.shape[1]
    d = plan.d
    ld = partial_ld(d)
    if dest is None:
        out = device_f64((d, n + 1), fortran=True, ld=ld)
        base, col_n = out, out[:, n]
    else:
        out, base, col_n = None, int(dest), int(dest) + 8 * ld * n
    st = current_stream()
    if plan.kind == "countsketch":
        plan.device_plan().apply(A_local, m_loc, n, lda, b_local, base, ld, col_n, partitions=1)
    elif plan.kind == "srht":
        words = plan.device_srht_words()
        _, sample = plan.op.device_srht()
        for src, ncol, ldsrc, dst in ((A_local, n, lda, base), (b_local, 1, m_loc, col_n)):
            _native.call("skl_srht_dense_shard", _native.ptr(src), m_loc, ncol, ldsrc,
                         _native.ptr(words), _native.ptr(sample), plan.op.padded_dim, d, plan.r0,
                         _native.ptr(dst), ld, st)
    else:
        G, ldg = plan.op.device_gaussian()
        Gs = G[:, plan.r0:]
        for src, ncol, ldsrc, dst in ((A_local, n, lda, base), (b_local, 1, m_loc, col_n)):
            _native.call("skl_gemm_f64", _native.ptr(Gs), ldg, _native.ptr(src), ldsrc,
                         _native.ptr(dst), ld, d, ncol, m_loc, 0, st)
    return out


class PeerSlots:
    """Fused reduce of the per-rank partials through NVLink peer memory.

    Every rank owns a symmetric buffer of 2 x world slots of ``rows x cols``
    (column-major, ld ``partial_ld(rows)``); rank r's sketch kernels write
    their partial into slot r of the destination rank's buffer
    (``slot_ptr()``, double-buffered by step parity), ``finish()`` runs the
    device-side barrier and, on the destination, the fixed-order slot sum.
    The parity buffers make one barrier per step enough: a rank rewrites a
    slot two steps later, after the barrier that follows the destination's
    previous sum.  ``timeout_ms`` turns a missing peer into an error instead
    of a hang."""

    def __init__(self, rows: int, cols: int, group=None, dst: int = 0, timeout_ms: int = 60000):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        require_cuda()
        self.group = group if group is not None else dist.group.WORLD
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.rows, self.cols, self.ld = rows, cols, partial_ld(rows)
        self.slot = cols * self.ld  # elements per slot
        self.dst, self.timeout_ms, self.step = dst, timeout_ms, 0
        self.buf = symm_mem.empty(2 * self.world * self.slot, dtype=torch.float64, device="cuda")
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        self.dst_base = int(self.hdl.buffer_ptrs[dst])

    def slot_ptr(self) -> int:
        """Device address of this rank's slot (current step) on the destination."""
        half = (self.step & 1) * self.world * self.slot
        return self.dst_base + 8 * (half + self.rank * self.slot)

    def finish(self, out=None, ldo: int = 0):
        """Barrier over the ranks' slot writes; on the destination the slots are
        summed in rank order into ``out`` (rows x cols, ld ``ldo``; None: the
        barrier only)."""
        self.hdl.barrier(channel=0, timeout_ms=self.timeout_ms)
        if self.rank == self.dst and out is not None:
            half = (self.step & 1) * self.world * self.slot
            _native.call("skl_sum_slots", self.buf.data_ptr() + 8 * half, self.world, self.slot,
                         self.rows, self.cols, self.ld, _native.ptr(out), ldo, current_stream())
        self.step += 1
        return out


def peer_slots_or_none(rows: int, cols: int, group=None, dst: int = 0):
    """PeerSlots when symmetric memory can be set up on this job, else None
    (the caller then falls back to a collective reduce)."""
    try:
        return PeerSlots(rows, cols, group, dst)
    except Exception:  # noqa: BLE001 - no symmetric memory: collective fallback
        return None


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
                             residual_local=None, collective: str = "auto"):
    """SAA over row-sharded data.  Returns (x, residual_norm, d) on every rank.

    ``local_apply(plan, A_local, b_local) -> partial`` defaults to the CUDA
    kernel; ``solve_reduced(partial) -> x`` and ``residual_local(A, b, x)``
    default to the device QR / residual kernels.  The hooks exist so the
    host-side sharding and collective logic can be exercised on CPU (gloo).
    ``collective``: "peer" (kernels write into rank 0's symmetric slots,
    fixed-order sum), "reduce" (one collective reduce), or "auto" (peer when
    the device path and symmetric memory are available).
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    r0, r1 = shard_rows(m_total, world, rank)
    if A_local.shape[0] != r1 - r0:
        raise ValueError(f"rank {rank} holds {A_local.shape[0]} rows, expected {r1 - r0}")
    op = build_sketch(spec, m_total)
    plan = ShardPlan(op, r0, r1)
    n = A_local.shape[1]
    d = plan.d
    slots = None
    if local_apply is None and collective in ("auto", "peer"):
        slots = PeerSlots(d, n + 1, group) if collective == "peer" else peer_slots_or_none(
            d, n + 1, group)
    if slots is not None:
        lda = int(A_local.stride(1)) if n > 1 else A_local.shape[0]
        local_partial_device(plan, A_local, lda, b_local, dest=slots.slot_ptr())
        partial = device_f64((d, n + 1), fortran=True, ld=partial_ld(d))
        slots.finish(partial, partial_ld(d))
    else:
        if local_apply is None:
            lda = int(A_local.stride(1)) if n > 1 else A_local.shape[0]
            partial = local_partial_device(plan, A_local, lda, b_local)
        else:
            partial = local_apply(plan, A_local, b_local)
        reduce_partials(partial, dist, group)
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
