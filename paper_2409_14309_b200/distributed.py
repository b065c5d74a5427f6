"""Row-sharded sketch-and-apply across GPUs.

Row block k of A (and b) lives on rank k.  Every rank sketches its block
with the operator realised once for the GLOBAL m, exactly as the reference
would build it (sketch.py:84-127) -- CountSketch hashes of global rows,
SRHT sign/sample with the shard's block offset, the Gaussian column block --
producing a partial d x (n+1) [SA | Sb].  Dense and CSR row blocks are both
supported (a CSR block is the rows [r0, r1) of the global CSR with its
indptr rebased; CountSketch uses the CSR kernel with the bucket lists of the
shard's rows, SRHT / Gaussian densify the block on the device as the
reference densifies CSR input, sketch.py:205-206, 214).

The reduce runs over NVLink peer memory (``PeerReduce``): every rank's
kernels write the partial into the rank's own symmetric buffer; after a
device-side barrier rank r sums element block r of all N partials in rank
order (loads from the peers' buffers) and stores it straight into the
destination's result buffer; a second barrier publishes the result.  That
is a reduce-scatter whose gather is the destination's inbox: each rank
moves ~(N-1)/N of one partial in and 1/N out (config 4's 64 MiB partial:
~56 MiB per rank, instead of the destination pulling N x 64 MiB), and the
sum is deterministic for a given world size.  Where symmetric memory is
unavailable (or on CPU with gloo, in the tests) the partials are combined by
one collective reduce instead.  The destination solves the reduced problem,
broadcasts x, and the residual norm is an all-reduce of the per-block
squared residuals.

The sum over ranks changes the floating-point order relative to the
single-pass fold, so the result is within ~1e-15 relative of the 1-GPU
(bitwise-reference) sketch, not bitwise.  Process layout: one process per
GPU, launched by torchrun (``launch.py``); ``torch.distributed`` is the
plumbing (process group, symmetric-memory rendezvous, broadcast).  The same
shard plans drive the single-process multi-device ``solve()``
(``multidevice.py``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
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


def element_block(total: int, world: int, rank: int, align: int = 2) -> tuple[int, int]:
    """Rank ``rank``'s share [e0, e1) of ``total`` flat elements in the
    reduce-scatter (block starts on multiples of ``align`` so 16-byte loads
    stay aligned; the blocks tile [0, total))."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    units = math.ceil(total / align)
    u0, u1 = units * rank // world, units * (rank + 1) // world
    return min(total, u0 * align), min(total, u1 * align)


def band_pieces(t0: int, t1: int, m: int, r0: int, r1: int):
    """The rectangles of S (row-major d x m, normal t at [t // m, t % m])
    that a band holding normals [t0, t1) contributes to the column block
    [r0, r1): [(row_begin, row_end, col_begin, col_end)] -- the band's
    partial first row, its full rows, its partial last row."""
    if t1 <= t0:
        return []
    i_first, i_last = t0 // m, (t1 - 1) // m
    rects = []
    for i in sorted({i_first, i_last}):
        rects.append((i, i + 1, max(0, t0 - i * m), min(m, t1 - i * m)))
    if i_last - i_first >= 2:
        rects.append((i_first + 1, i_last, 0, m))
    out = []
    for ia, ib, lo, hi in rects:
        a, c = max(lo, r0), min(hi, r1)
        if a < c and ia < ib:
            out.append((ia, ib, a, c))
    return out


def band_bounds(N: int, world: int, seg_words: int) -> list[int]:
    """Segment boundaries of the N-normal stream's bands (~1.025 words per
    normal: 3 % slack, as the one-device generator)."""
    seg_total = int(N * 1.03 / seg_words) + 8
    return [seg_total * k // world for k in range(world + 1)]


@dataclass(frozen=True)
class CsrBlock:
    """Rows [r0, r1) of a CSR matrix on one device: indptr rebased to 0
    (int64), the block's int64 column indices and float64 values."""

    indptr: object
    indices: object
    values: object
    rows: int
    cols: int

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def dense(self):
        """Column-major m_loc x n dense copy on the device (the reference
        densifies CSR input for SRHT / Gaussian, sketch.py:205-206, 214)."""
        rows = torch.repeat_interleave(torch.arange(self.rows, device=self.indptr.device),
                                       self.indptr[1:] - self.indptr[:-1])
        out = torch.zeros((self.cols, self.rows), dtype=torch.float64, device=self.indptr.device)
        out[self.indices, rows] = self.values
        return out.t()


def csr_row_block(A, r0: int, r1: int, device=None) -> CsrBlock:
    """Rows [r0, r1) of a SparseMatrix (or scipy CSR) as a CsrBlock on
    ``device`` (a CUDA index, default the current device, or a torch device)."""
    if hasattr(A, "values"):  # SparseMatrix carrier (linalg.py:56-114)
        vals, ncols = A.values, A.cols
    else:  # scipy.sparse CSR
        vals, ncols = A.data, A.shape[1]
    indptr = np.asarray(A.indptr, dtype=np.int64)
    p0, p1 = int(indptr[r0]), int(indptr[r1])
    if isinstance(device, (str, torch.device)):
        dev = torch.device(device)  # e.g. "cpu" for the gloo tests' oracle ranks
    else:
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    def up(a, dtype):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(dev)

    return CsrBlock(up(indptr[r0:r1 + 1] - p0, np.int64), up(np.asarray(A.indices)[p0:p1], np.int64),
                    up(np.asarray(vals)[p0:p1], np.float64), r1 - r0, int(ncols))


class ShardPlan:
    """The part of a global operator that the rank owning rows [r0, r1) needs.

    * countsketch: the hashes/signs of the global rows [r0, r1), their dense
      plan and (for CSR blocks and vector applies) their bucket lists -- the
      hash of row j is the reference's draw for GLOBAL j; the device hashes
      are drawn on the shard's device from the operator's key;
    * srht: the packed sign words of the shard's 4096-row blocks (a slice of
      the global packing, shards are block aligned) plus the global sample;
      the kernel adds the (-1)^popc(p_hi & j_hi) factor for the shard's
      block offset, i.e. H_m = H_G (x) H_{m/G} over (shard, local) bits;
    * gaussian: the column block S[:, r0:r1] of the row-major d x m matrix
      (``op.device_gaussian_block``: on a multi-device run each device
      generates only its band of the stream and the blocks are exchanged)."""

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
        self._dev: dict = {}
        # (G block, ld) supplied by a banded multi-device generation
        # (multidevice.gaussian_column_blocks); None: slice the full G
        self.gaussian_block = None

    @property
    def rows(self):
        return np.ascontiguousarray(self.op.rows[self.r0:self.r1])

    @property
    def signs(self):
        return np.ascontiguousarray(self.op.signs[self.r0:self.r1])

    def _cache(self) -> dict:
        return self._dev.setdefault(torch.cuda.current_device(), {})

    def device_hashes(self):
        """(rows int32, signs int8) of the shard's rows on the current device."""
        c = self._cache()
        if "hash" not in c:
            r, s = self.op.device_hashes()
            c["hash"] = (r[self.r0:self.r1], s[self.r0:self.r1])
        return c["hash"]

    def device_plan(self) -> CountSketchPlan:
        c = self._cache()
        if "plan" not in c:
            m_loc = self.r1 - self.r0
            if torch.cuda.is_available() and _native.plan_geometry(self.d)[0] == "owned":
                h = self.device_hashes()
                c["plan"] = CountSketchPlan.from_device(h[0], h[1], self.d, m_loc)
            else:
                c["plan"] = CountSketchPlan(self.rows, self.signs, self.d)
        return c["plan"]

    def device_buckets(self):
        """(bucket_rows int32 local, bucket_ptr int64, bucket-ordered signs)
        of the shard's rows: the CSR of S[:, r0:r1] (within a bucket the rows
        stay ascending -- the stable sort of the shard's hashes)."""
        c = self._cache()
        if "buckets" not in c:
            rows_d, signs_d = self.device_hashes()
            order = torch.sort(rows_d, stable=True).indices
            bptr = torch.zeros(self.d + 1, dtype=torch.int64, device=rows_d.device)
            bptr[1:] = torch.cumsum(torch.bincount(rows_d, minlength=self.d), 0)
            c["buckets"] = (order.to(torch.int32), bptr, signs_d[order].contiguous())
        return c["buckets"]

    def device_srht_words(self):
        """Packed sign words of this shard's blocks (device view)."""
        signs, _ = self.op.device_srht()
        B = min(self.op.padded_dim, 4096)
        per_block = int(_native.lib().skl_srht_sign_words(B))
        return signs[(self.r0 // B) * per_block:]

    def device_gaussian(self):
        """(G block view d x (r1 - r0), ld) on the current device."""
        if self.gaussian_block is not None:
            return self.gaussian_block
        G, ldg = self.op.device_gaussian_block(self.r0, self.r1)
        return G, ldg


def partial_ld(d: int) -> int:
    """Leading dimension of a d x (n+1) partial (keeps the Sb column 16-byte
    aligned)."""
    return (d + 1) // 2 * 2


def local_partial_device(plan: ShardPlan, A_local, lda: int, b_local, dest: int | None = None):
    """Partial [SA | Sb] of one row block on this rank's GPU: a d x (n+1)
    column-major tensor (ld ``partial_ld(d)``) whose last column is the
    partial Sb.  ``A_local`` is a dense column-major tensor (ld ``lda``) or a
    CsrBlock.  With ``dest`` (a device address, e.g. this rank's symmetric
    buffer) the kernels write there instead and None is returned."""
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
    if isinstance(A_local, CsrBlock):
        if plan.kind == "countsketch":
            brow, bptr, bsign = plan.device_buckets()
            _native.call("skl_countsketch_csr", _native.ptr(A_local.indptr),
                         _native.ptr(A_local.indices), _native.ptr(A_local.values), m_loc, n,
                         _native.ptr(brow), _native.ptr(bptr), _native.ptr(bsign), d,
                         _native.ptr(base), ld, st)
            _native.call("skl_countsketch_dense_ordered", None, m_loc, 0, m_loc,
                         _native.ptr(b_local), _native.ptr(brow), _native.ptr(bptr),
                         _native.ptr(bsign), 1.0, d, None, ld, _native.ptr(col_n), 0, st)
            return out
        A_local = A_local.dense()
        lda = m_loc
    if plan.kind == "countsketch":
        plan.device_plan().apply(A_local, m_loc, n, lda, b_local, base, ld, col_n, partitions=1)
    elif plan.kind == "srht":
        # [A | b] of the shard in one pass, b as the last column
        words = plan.device_srht_words()
        _, sample = plan.op.device_srht()
        _native.call("skl_srht_dense_ab", _native.ptr(A_local), m_loc, n, lda, _native.ptr(b_local),
                     _native.ptr(words), _native.ptr(sample), plan.op.padded_dim, d, plan.r0,
                     _native.ptr(base), ld, _native.ptr(col_n), 1, st)
    else:
        Gs, ldg = plan.device_gaussian()
        for src, ncol, ldsrc, dst in ((A_local, n, lda, base), (b_local, 1, m_loc, col_n)):
            _native.call("skl_gemm_f64", _native.ptr(Gs), ldg, _native.ptr(src), ldsrc,
                         _native.ptr(dst), ld, d, ncol, m_loc, 0, st)
    return out


class PeerReduce:
    """Reduce of the per-rank partials over NVLink peer memory.

    Every rank owns a symmetric buffer [partial | result] of ``rows x cols``
    each (column-major, ld ``partial_ld(rows)``).  A rank's sketch kernels
    write into ``partial_ptr()`` (its own buffer); ``finish()`` runs a
    device-side barrier, reduces this rank's element block of all partials
    in rank order into the destination's result buffer (skl_reduce_peers:
    peer loads, peer stores), and a second barrier publishes the result.
    Two barriers per step also make one partial buffer enough: no rank
    rewrites its partial before every rank has finished reading it.
    ``timeout_ms`` turns a missing peer into an error instead of a hang."""

    def __init__(self, rows: int, cols: int, group=None, dst: int = 0, timeout_ms: int = 60000):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        require_cuda()
        self.group = group if group is not None else dist.group.WORLD
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 16:
            raise ValueError("PeerReduce supports up to 16 ranks")
        self.rows, self.cols, self.ld = rows, cols, partial_ld(rows)
        self.slot = cols * self.ld  # elements per partial
        self.dst, self.timeout_ms = dst, timeout_ms
        enable = getattr(symm_mem, "enable_symm_mem_for_group", None)
        if enable is not None:  # idempotent; required before rendezvous on some versions
            enable(self.group.group_name)
        self.buf = symm_mem.empty(2 * self.slot, dtype=torch.float64, device="cuda")
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        self.peers = [int(p) for p in self.hdl.buffer_ptrs]
        self.e0, self.e1 = element_block(self.slot, self.world, self.rank)
        self._peer_arr = _native.ptr_array(self.peers)

    def partial_ptr(self) -> int:
        """Device address of this rank's partial (its own buffer)."""
        return self.peers[self.rank]

    def result_view(self):
        """The reduced rows x cols result (column-major view) on the destination."""
        r = self.buf[self.slot:].view(self.cols, self.ld).t()
        return r[: self.rows]

    def finish(self, out=None, ldo: int = 0):
        """Barrier, this rank's block of the fixed-order sum into the
        destination's result, barrier.  On the destination the result is
        copied into ``out`` (rows x cols, ld ``ldo``) when given; returns the
        result view there (None elsewhere)."""
        self.hdl.barrier(channel=0, timeout_ms=self.timeout_ms)
        _native.call("skl_reduce_peers", self._peer_arr, self.world, self.e0, self.e1,
                     self.peers[self.dst] + 8 * self.slot, current_stream())
        self.hdl.barrier(channel=0, timeout_ms=self.timeout_ms)
        if self.rank != self.dst:
            return None
        res = self.result_view()
        if out is not None:
            out.copy_(res)
        return res


def peer_reduce_or_none(rows: int, cols: int, group=None, dst: int = 0):
    """PeerReduce when symmetric memory can be set up on this job, else None
    (the caller then falls back to a collective reduce)."""
    try:
        return PeerReduce(rows, cols, group, dst)
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


def residual_sq_local(A_local, lda: int, b_local, x) -> float:
    """||A_local x - b_local||^2 of one row block (dense or CsrBlock) on its
    device (the reference's _residual_norm, solvers.py:102-107, per block)."""
    out = np.zeros(1)
    st = current_stream()
    if isinstance(A_local, CsrBlock):
        _native.call("skl_residual_csr", _native.ptr(A_local.indptr), _native.ptr(A_local.indices),
                     _native.ptr(A_local.values), A_local.rows, A_local.cols, _native.ptr(x),
                     _native.ptr(b_local), _native.ptr(out), st)
    else:
        _native.call("skl_residual_dense", _native.ptr(A_local), A_local.shape[0],
                     A_local.shape[1], lda, _native.ptr(x), _native.ptr(b_local),
                     _native.ptr(out), st)
    return float(out[0]) ** 2


def exchange_gaussian_bands(band, t0: int, t1: int, all_t, m: int, d: int, spans, rank: int,
                            dist, group=None, device=None):
    """All-to-all of the Gaussian operator's bands (multi-process form of
    multidevice.gaussian_column_blocks): this rank holds normals [t0, t1)
    (``band``: rows t0 // m .. of S, row-major, any ld; None when empty),
    ``all_t`` every rank's range, ``spans`` every rank's row shard.  Each
    rank sends every other rank the rectangles of its band inside that
    rank's column block (band_pieces), packed in order; the receiver
    unpacks them with the same rectangles computed from the sender's range.
    Returns this rank's block S[:, r0:r1] (d x w tensor, ld rounded to 32)."""
    world = len(spans)
    r0, r1 = spans[rank]
    w = r1 - r0
    ldb = (w + 31) // 32 * 32
    dev = device if device is not None else (band.device if band is not None else "cpu")
    blk = torch.zeros((d, ldb), dtype=torch.float64, device=dev)
    row0 = t0 // m
    send = []
    for s in range(world):
        ps = band_pieces(t0, t1, m, *spans[s]) if band is not None else []
        send.append([band[ia - row0:ib - row0, a:c].reshape(-1) for ia, ib, a, c in ps])
    in_sizes = [sum(p.numel() for p in parts) for parts in send]
    recv_pieces = [band_pieces(tk0, tk1, m, r0, r1) for tk0, tk1 in all_t]
    out_sizes = [sum((ib - ia) * (c - a) for ia, ib, a, c in ps) for ps in recv_pieces]
    flat = [p for parts in send for p in parts]
    sendbuf = (torch.cat(flat) if flat else torch.zeros(0, dtype=torch.float64, device=dev))
    recvbuf = torch.empty(sum(out_sizes), dtype=torch.float64, device=dev)
    dist.all_to_all_single(recvbuf, sendbuf, out_sizes, in_sizes, group=group)
    off = 0
    for ps in recv_pieces:
        for ia, ib, a, c in ps:
            nel = (ib - ia) * (c - a)
            blk[ia:ib, a - r0:c - r0] = recvbuf[off:off + nel].view(ib - ia, c - a)
            off += nel
    return blk, ldb


def gaussian_block_distributed(op, spans, dist, group=None):
    """This rank's Gaussian column block, generated in bands across the ranks
    (skl_gaussian_band_*: each rank parses ~1/N of the stream; the bands'
    normal counts are all-gathered, then exchange_gaussian_bands)."""
    import ctypes

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    _native.install_gaussian_tables()
    lib = _native.lib()
    d, m = op.target_dim, op.source_dim
    N = d * m
    bounds = band_bounds(N, world, int(lib.skl_gaussian_segment_words()))
    st = current_stream()

    def begin(seg0, seg1):
        h = ctypes.c_void_p()
        _native.call("skl_gaussian_band_begin", op.key, seg0, seg1, ctypes.byref(h), None, st)
        c = ctypes.c_int64()
        _native.call("skl_gaussian_band_count", h, ctypes.byref(c), st)
        return h, int(c.value)

    h, cnt = begin(bounds[rank], bounds[rank + 1])
    while True:
        counts = torch.zeros(world, dtype=torch.int64, device="cuda")
        counts[rank] = cnt
        dist.all_reduce(counts, group=group)
        counts = [int(v) for v in counts.cpu()]
        if sum(counts) >= N:
            break
        if rank == world - 1:  # too few words: the last band grows
            lib.skl_gaussian_band_free(h, ctypes.c_void_p(st))
        bounds[-1] += (bounds[-1] - bounds[-2]) // 8 + 16
        if rank == world - 1:
            h, cnt = begin(bounds[-2], bounds[-1])
    firsts = [sum(counts[:k]) for k in range(world)]
    all_t = [(min(N, firsts[k]), min(N, firsts[k] + counts[k])) for k in range(world)]
    t0, t1 = all_t[rank]
    band = None
    if t1 > t0:
        ldg = (m + 31) // 32 * 32
        band = torch.empty(((t1 - 1) // m + 1 - t0 // m, ldg), dtype=torch.float64, device="cuda")
        _native.call("skl_gaussian_band_write", h, firsts[rank], N, m, t0 // m,
                     _native.ptr(band), ldg, math.sqrt(d), st)
    else:
        lib.skl_gaussian_band_free(h, ctypes.c_void_p(st))
    return exchange_gaussian_bands(band, t0, t1, all_t, m, d, spans, rank, dist, group,
                                   device=torch.device("cuda", torch.cuda.current_device()))


def sharded_sketch_and_apply(A_local, b_local, m_total: int, spec, dist, group=None,
                             local_apply: Callable | None = None, solve_reduced=None,
                             residual_local=None, collective: str = "auto"):
    """SAA over row-sharded data.  Returns (x, residual_norm, d) on every rank.

    ``A_local`` is this rank's row block: a dense column-major tensor or a
    CsrBlock.  ``local_apply(plan, A_local, b_local) -> partial`` defaults to
    the CUDA kernels; ``solve_reduced(partial) -> x`` and
    ``residual_local(A, b, x)`` default to the device QR / residual kernels.
    The hooks exist so the host-side sharding and collective logic can be
    exercised on CPU (gloo).  ``collective``: "peer" (PeerReduce over
    symmetric memory), "reduce" (one collective reduce), or "auto" (peer
    when the device path and symmetric memory are available).
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    r0, r1 = shard_rows(m_total, world, rank)
    if A_local.shape[0] != r1 - r0:
        raise ValueError(f"rank {rank} holds {A_local.shape[0]} rows, expected {r1 - r0}")
    op = build_sketch(spec, m_total)
    plan = ShardPlan(op, r0, r1)
    if op.kind == "gaussian" and local_apply is None and world > 1:
        # the operator in bands across the ranks, not all of G on every rank
        key = ("gauss_dist", world, rank)
        if key not in op._host:
            spans = [shard_rows(m_total, world, k) for k in range(world)]
            op._host[key] = gaussian_block_distributed(op, spans, dist, group)
        plan.gaussian_block = op._host[key]
    n = A_local.shape[1]
    d = plan.d
    dense = not isinstance(A_local, CsrBlock)
    lda = (int(A_local.stride(1)) if n > 1 else A_local.shape[0]) if dense else 0
    peer = None
    if local_apply is None and collective in ("auto", "peer"):
        peer = PeerReduce(d, n + 1, group) if collective == "peer" else peer_reduce_or_none(
            d, n + 1, group)
    if peer is not None:
        local_partial_device(plan, A_local, lda, b_local, dest=peer.partial_ptr())
        partial = peer.finish()
    else:
        if local_apply is None:
            partial = local_partial_device(plan, A_local, lda, b_local)
        else:
            partial = local_apply(plan, A_local, b_local)
        reduce_partials(partial, dist, group)
    if rank == 0:
        if solve_reduced is None:
            from .linalg import reduced_solve_device

            x = reduced_solve_device(partial[:, :n], int(partial.stride(1)), partial[:, n], d, n)
        else:
            x = solve_reduced(partial)
    else:
        x = torch.empty(n, dtype=torch.float64,
                        device=b_local.device if hasattr(b_local, "device") else "cpu")
    dist.broadcast(x, src=0, group=group)
    if residual_local is None:
        r2 = torch.tensor([residual_sq_local(A_local, lda, b_local, x)], dtype=torch.float64,
                          device=x.device)
    else:
        r2 = residual_local(A_local, b_local, x)
    dist.all_reduce(r2, op=dist.ReduceOp.SUM, group=group)
    return x, float(torch.sqrt(r2).item()), d
