"""Sketching operators on the B200 engine.

Public surface and semantics follow /root/reference/pkg/src/sketchls/sketch.py
(`KINDS` :31-32, `default_embed_dim` :41-45, `SketchSpec` :48-63,
`SketchOperator` :66-81, `build_sketch` :84-127, `apply_to_matrix` :180-188,
`apply_to_vector` :191-195, `_apply` :198-223, `materialize` :226-242).

What changes is where the work runs:

* the seeded draws (bucket hashes, signs, SRHT sign diagonal and row sample)
  come from the native bit-exact Philox generator (``_native``), identical
  to what numpy 2.3.5 produces for the reference;
* a CountSketch operator keeps its hashes (not a scipy CSR) plus a chunked,
  bucket-sorted *plan* cached on the device; the apply is the
  ``skl_countsketch_dense`` kernel (bitwise-equal to scipy's
  ``csr_matvecs`` fold) or the CSR scatter kernel;
* SRHT and Gaussian applies run in their own sm_100a kernels.

There is no host fallback: without the CUDA library the applies raise.
"""

from __future__ import annotations

import math
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from . import _native
from ._device import current_stream, device_f64, require_cuda, to_device, torch
from .errors import CapacityError, ShapeError, SpecError
from .linalg import DenseMatrix, Matrix, SparseMatrix, Vector, _freeze
from .rng import derive_seed, stream

KINDS = ("gaussian", "srht", "countsketch", "sparsesign", "identity")
DEFAULT_KIND = "countsketch"
# Kinds with a native implementation in this engine.
ENGINE_KINDS = ("gaussian", "srht", "countsketch", "sparsesign", "identity")

# Chunk bound (entries) of the dense key matrix when sampling distinct rows in
# the collision-prone regime (sketch.py:35).
_SAMPLE_CHUNK_ENTRIES = 5 * 10**7

_MATERIALIZE_GUARD = 10**7

# Row-shard boundaries (distributed.shard_rows) are multiples of this.
SHARD_ALIGN = 8192
# Shared memory per CTA available to the apply kernels' rings.
_SMEM_BUDGET = 226 * 1024


class CountSketchPlan:
    """Device form of a CountSketch's hashes for the dense apply kernels.

    kind "owned" (d <= 4096): each bucket's running sum lives in a register
    of one lane for the whole apply (skl_countsketch_dense_owned);
    kind "lanes" (larger d): shared-memory accumulators fed by per-lane
    lists (skl_countsketch_dense).  Either way the per-bucket fold order is
    ascending source row, so the ordered apply is bitwise-equal to scipy."""

    def __init__(self, rows: np.ndarray, signs: np.ndarray, d: int, kind: str | None = None,
                 spr: int = 1):
        self.d = int(d)
        self.spr = int(spr)
        self.scale = 1.0 / math.sqrt(spr) if spr > 1 else 1.0
        self.kind, self.chunk, self.warps = _native.plan_geometry(
            self.d, kind, m=None if spr > 1 else int(np.asarray(signs).shape[0]))
        if spr > 1:
            if self.kind == "owned":  # the owned plan's 13-bit row field counts entries
                self.chunk = max(8, self.chunk // spr // 8 * 8)
            rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(-1)
            signs = np.ascontiguousarray(signs, dtype=np.int8).reshape(-1)
        # The kernels' ring stages (A chunk + plan block) must fit shared
        # memory: shrink the chunk when few buckets make per-lane lists long.
        while True:
            if self.kind == "owned":
                lanes, off, mx = _native.countsketch_plan_owned(rows, signs, self.d, self.chunk,
                                                                self.warps, spr=self.spr)
                need = 2 * ((self.chunk + 2) * 8 + 2 * mx + 127)
            else:
                lanes, off, mx = _native.countsketch_plan(rows, signs, self.d, self.chunk,
                                                          self.warps, spr=self.spr)
                need = 3 * ((self.chunk + 2) * 8 + 4 * mx + 127) + (self.d + 1) * 8 + 256
            if need <= _SMEM_BUDGET or self.chunk <= 8:
                break
            self.chunk = max(8, int(self.chunk * 0.9 * _SMEM_BUDGET / need) // 8 * 8)
        self.lanes = to_device(lanes.view(np.int16 if self.kind == "owned" else np.int32))
        self.off = to_device(off)
        self.max_block = mx
        self.plan_bytes = int(lanes.nbytes + off.nbytes)

    @classmethod
    def from_device(cls, rows_d, signs_d, d: int, m: int) -> "CountSketchPlan":
        """Register-owned plan built on the device from device hashes
        (skl_countsketch_plan_owned_device: the same words as the host)."""
        self = cls.__new__(cls)
        self.d = int(d)
        self.spr, self.scale = 1, 1.0
        self.kind, self.chunk, self.warps = _native.plan_geometry(self.d, "owned", m=m)
        st = current_stream()
        tm = np.zeros(2, dtype=np.int64)
        while True:
            nch = (m + self.chunk - 1) // self.chunk
            off = torch.empty(nch + 1, dtype=torch.int64, device="cuda")
            maxlen = torch.empty(nch * self.warps, dtype=torch.int32, device="cuda")
            _native.call("skl_countsketch_plan_owned_device", _native.ptr(rows_d),
                         _native.ptr(signs_d), m, self.d, self.chunk, self.warps, None,
                         _native.ptr(off), _native.ptr(maxlen), _native.ptr(tm), st)
            mx = int(tm[1])
            need = 2 * ((self.chunk + 2) * 8 + 2 * mx + 127)
            if need <= _SMEM_BUDGET or self.chunk <= 8:
                break
            self.chunk = max(8, int(self.chunk * 0.9 * _SMEM_BUDGET / need) // 8 * 8)
        lanes = torch.empty(max(int(tm[0]), 8), dtype=torch.int16, device="cuda")
        _native.call("skl_countsketch_plan_owned_device", _native.ptr(rows_d),
                     _native.ptr(signs_d), m, self.d, self.chunk, self.warps, _native.ptr(lanes),
                     _native.ptr(off), _native.ptr(maxlen), None, st)
        self.lanes, self.off, self.max_block = lanes, off, mx
        self.plan_bytes = int(tm[0]) * 2 + (nch + 1) * 8
        return self

    def apply(self, A, m: int, n: int, lda: int, b, out, ldo: int, outb,
              partitions: int = 0, accumulate: int = 0, stream=None) -> None:
        """out[:, :n] (+)= S A, outb (+)= S b on the device (raw pointers or tensors)."""
        if getattr(self, "spr", 1) > 1:
            fn = "skl_sparsesign_dense_owned" if self.kind == "owned" else "skl_sparsesign_dense"
            _native.call(fn, _native.ptr(A), m, n, lda, _native.ptr(b),
                         _native.ptr(self.lanes), _native.ptr(self.off), self.max_block, self.d,
                         self.chunk, self.warps, self.scale, _native.ptr(out), ldo,
                         _native.ptr(outb), partitions, accumulate,
                         current_stream() if stream is None else stream)
            return
        fn = "skl_countsketch_dense_owned" if self.kind == "owned" else "skl_countsketch_dense"
        _native.call(fn, _native.ptr(A), m, n, lda, _native.ptr(b), _native.ptr(self.lanes),
                     _native.ptr(self.off), self.max_block, self.d, self.chunk, self.warps,
                     _native.ptr(out), ldo, _native.ptr(outb), partitions, accumulate,
                     current_stream() if stream is None else stream)

    def apply_host(self, A, m: int, n: int, lda: int, b, SA, ldsa: int, Sb,
                   A_keep=None, ld_keep: int = 0, b_keep=None, stream=None) -> None:
        """Host A/b in, host SA/Sb out; H2D streamed under the kernel."""
        fn = ("skl_countsketch_dense_owned_host" if self.kind == "owned"
              else "skl_countsketch_dense_host")
        _native.call(fn, _native.ptr(A), m, n, lda, _native.ptr(b), _native.ptr(self.lanes),
                     _native.ptr(self.off), self.max_block, self.d, self.chunk, self.warps,
                     _native.ptr(SA), ldsa, _native.ptr(Sb), _native.ptr(A_keep), ld_keep,
                     _native.ptr(b_keep), current_stream() if stream is None else stream)


def default_embed_dim(m: int, n: int, d_factor: float = 4.0) -> int:
    """ceil(d_factor*n) clamped to [n, m] (sketch.py:41-45)."""
    return min(m, max(n, math.ceil(d_factor * n)))


@dataclass(frozen=True)
class SketchSpec:
    """Declarative description of a sketching map (sketch.py:48-63)."""

    kind: str
    embed_dim: int
    seed: int = 0
    sparsity: int = 8

    def __post_init__(self) -> None:
        if self.kind not in KINDS:
            raise SpecError(f"unknown sketch kind {self.kind!r}, expected one of {KINDS}")
        if self.embed_dim < 1:
            raise SpecError(f"embed_dim must be >= 1, got {self.embed_dim}")
        if self.kind == "sparsesign" and self.sparsity < 1:
            raise SpecError(f"sparsity must be >= 1, got {self.sparsity}")


class SketchOperator:
    """A seeded realisation of a sketch for one source dimension.

    Immutable; rebuilding with the same (spec, m) reproduces it bitwise.
    Besides the reference's fields it keeps the raw CountSketch hashes
    (``rows`` int32, ``signs`` int8) and per-device caches of what the
    kernels consume.  ``sparse_map`` / ``gaussian_entries`` are built on
    demand for compatibility with code that inspects them."""

    __slots__ = ("kind", "source_dim", "target_dim", "_rows", "_signs", "sign_diag",
                 "row_sample", "padded_dim", "key", "sparsity", "_dev", "_host", "_lock")

    def __init__(self, kind, source_dim, target_dim, rows=None, signs=None, sign_diag=None,
                 row_sample=None, padded_dim=None, key=None, device_hashes=None, sparsity=None):
        for name, val in (("kind", kind), ("source_dim", source_dim),
                          ("target_dim", target_dim), ("_rows", rows), ("_signs", signs),
                          ("sign_diag", sign_diag), ("row_sample", row_sample),
                          ("padded_dim", padded_dim), ("key", key), ("sparsity", sparsity)):
            object.__setattr__(self, name, val)
        object.__setattr__(self, "_dev", {})
        object.__setattr__(self, "_host", {})
        object.__setattr__(self, "_lock", threading.RLock())
        if device_hashes is not None:
            with torch.cuda.device(device_hashes[0].device):
                self._cached("hash", lambda: device_hashes)

    # CountSketch hashes: built on the device when a GPU is present (see
    # _build_sketch); the host copies are fetched on first use.
    def _host_hashes(self):
        with self._lock:
            if "hash" not in self._host:
                for dev, c in list(self._dev.items()):
                    if "hash" in c:
                        with torch.cuda.device(dev):
                            r, g = self._cached("hash", None)
                            self._host["hash"] = (_freeze(r.cpu().numpy()),
                                                  _freeze(g.cpu().numpy()))
                        break
            return self._host.get("hash")

    @property
    def rows(self):
        if self._rows is None and self.kind == "countsketch":
            return self._host_hashes()[0]
        return self._rows

    @property
    def signs(self):
        if self._signs is None and self.kind == "countsketch":
            return self._host_hashes()[1]
        return self._signs

    def __setattr__(self, name, value):
        raise AttributeError("SketchOperator is immutable")

    def __repr__(self) -> str:
        return (f"SketchOperator(kind={self.kind!r}, source_dim={self.source_dim}, "
                f"target_dim={self.target_dim})")

    # ------------------------------------------------ reference-compatible views
    @property
    def sparse_map(self):
        """d x m scipy CSR of a CountSketch (sketch.py:100-102) or a sparse
        sign embedding (:110-114), built lazily."""
        if self.kind not in ("countsketch", "sparsesign"):
            return None
        if "csr" not in self._host:
            m, d = self.source_dim, self.target_dim
            if self.kind == "countsketch":
                vals = self.signs.astype(np.float64)
                rows, cols = self.rows.astype(np.int64), np.arange(m)
            else:
                s = self.sparsity
                vals = self.signs.astype(np.float64).ravel() / math.sqrt(s)
                rows, cols = self.rows.astype(np.int64).ravel(), np.repeat(np.arange(m), s)
            self._host["csr"] = scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(d, m),
                                                        dtype=np.float64)
        return self._host["csr"]

    @property
    def gaussian_entries(self):
        """d x m Gaussian entries (sketch.py:94-96), copied back from the device."""
        if self.kind != "gaussian":
            return None
        if "g" not in self._host:
            G, ldg = self.device_gaussian()
            host = G[:, : self.source_dim].cpu().numpy() if ldg != self.source_dim else G.cpu().numpy()
            self._host["g"] = _freeze(np.ascontiguousarray(host))
        return self._host["g"]

    # ------------------------------------------------------------ device caches
    # Per-device artifacts (hashes, plans, bucket lists, SRHT words, G) are
    # built once on the stream of the first caller and shared with callers
    # on any stream: each entry keeps the event recorded after its build,
    # every consumer's stream waits on it, and the tensors are recorded on
    # the consumer's stream so an evicted operator's memory is not reused
    # while a kernel on another stream still reads it.
    def _cache(self):
        dev = torch.cuda.current_device()
        with self._lock:
            return self._dev.setdefault(dev, {})

    def _cached(self, name: str, build):
        c = self._cache()
        with self._lock:
            entry = c.get(name)
            if entry is None:
                if build is None:
                    return None
                value = build()
                st0 = torch.cuda.current_stream()
                ev = torch.cuda.Event()
                ev.record(st0)
                entry = c[name] = (value, ev, st0.cuda_stream)
        value, ev, made_on = entry
        if current_stream() == made_on:
            # the stream that built it: stream order already covers the build
            # and the allocator's own bookkeeping the lifetime
            return value
        st = torch.cuda.current_stream()
        if torch.cuda.is_current_stream_capturing():
            # inside a CUDA-graph capture the artifact was built before the
            # capture began (the warm-up call); an event from outside the
            # capture cannot be waited on there
            return value
        st.wait_event(ev)
        for t in _tensors_of(value):
            t.record_stream(st)
        return value

    def device_plan(self) -> CountSketchPlan:
        """The CountSketch apply plan on the current device (built once; on
        the device from device hashes when they are there)."""
        require_cuda()

        def build():
            if self.kind == "sparsesign":
                # register-owned plan up to d = 4096, shared-memory lane lists beyond
                return CountSketchPlan(self.rows, self.signs, self.target_dim, spr=self.sparsity)
            d = self.target_dim
            if _native.plan_geometry(d)[0] == "owned":
                rows_d, signs_d = self.device_hashes()
                return CountSketchPlan.from_device(rows_d, signs_d, d, self.source_dim)
            return CountSketchPlan(self.rows, self.signs, d)

        return self._cached("plan", build)

    def device_hashes(self):
        """CountSketch hashes in row order on the current device: (rows int32,
        signs int8) -- drawn there from the operator's key (the device draw
        is bit-identical to the host walk), else uploaded once."""
        require_cuda()

        def build():
            if self.kind == "countsketch" and self.key is not None:
                m, d = self.source_dim, self.target_dim
                rows_d = torch.empty(m, dtype=torch.int32, device="cuda")
                signs_d = torch.empty(m, dtype=torch.int8, device="cuda")
                _native.call("skl_rng_countsketch_device", self.key, m, d, _native.ptr(rows_d),
                             _native.ptr(signs_d), current_stream())
                return rows_d, signs_d
            return (to_device(np.ascontiguousarray(self.rows, dtype=np.int32)),
                    to_device(np.ascontiguousarray(self.signs, dtype=np.int8)))

        return self._cached("hash", build)

    def device_buckets(self):
        """(bucket_rows int32, bucket_ptr int64, bucket-ordered signs int8) on
        the current device: the CSR of S consumed by the CSR-operand kernel
        and the ordered few-column walk (for a sparse sign embedding each
        source row appears in s buckets)."""
        require_cuda()

        def build():
            if self.kind == "countsketch":
                # stable sort of the row-order hashes by bucket, on the device
                rows_d, signs_d = self.device_hashes()
                order = torch.sort(rows_d, stable=True).indices
                bptr = torch.zeros(self.target_dim + 1, dtype=torch.int64, device=rows_d.device)
                bptr[1:] = torch.cumsum(torch.bincount(rows_d, minlength=self.target_dim), 0)
                return order.to(torch.int32), bptr, signs_d[order].contiguous()
            spr = self.sparsity if self.kind == "sparsesign" else 1
            flat_rows = np.ascontiguousarray(self.rows.reshape(-1), dtype=np.int32)
            ent, bptr = _native.countsketch_buckets(flat_rows, self.target_dim)
            bsign = np.ascontiguousarray(self.signs.reshape(-1)[ent])
            brow = (ent // spr).astype(np.int32) if spr > 1 else ent
            return to_device(brow), to_device(bptr), to_device(bsign)

        return self._cached("buckets", build)

    def device_srht(self):
        require_cuda()

        def build():
            signs8 = np.where(self.sign_diag > 0, 1, -1).astype(np.int8)
            return to_device(_native.srht_pack_signs(signs8)), to_device(self.row_sample)

        return self._cached("srht", build)

    def device_gaussian_block(self, r0: int, r1: int):
        """(G[:, r0:r1] view, ld) on the current device: the column block a
        row shard [r0, r1) of A multiplies."""
        G, ldg = self.device_gaussian()
        return G[:, r0:r1], ldg

    def device_gaussian(self):
        """G (d x m, row-major like numpy's C order, ld = ldg) on the device."""
        require_cuda()

        def build():
            d, m = self.target_dim, self.source_dim
            ldg = (m + 31) // 32 * 32
            G = torch.empty((d, ldg), dtype=torch.float64, device="cuda")
            _native.install_gaussian_tables()
            _native.call("skl_rng_gaussian_device", self.key, d, m, _native.ptr(G), ldg,
                         current_stream())
            return G, ldg

        return self._cached("gauss", build)


def _tensors_of(value):
    """The CUDA tensors inside a cached artifact (tensor, tuple, or plan)."""
    if torch is not None and isinstance(value, torch.Tensor):
        return (value,) if value.is_cuda else ()
    if isinstance(value, (tuple, list)):
        return tuple(t for v in value for t in _tensors_of(v))
    if isinstance(value, CountSketchPlan):
        return tuple(t for t in (value.lanes, value.off) if isinstance(t, torch.Tensor))
    return ()


_OP_CACHE: "OrderedDict[tuple, SketchOperator]" = OrderedDict()
_OP_CACHE_LOCK = threading.Lock()
OP_CACHE_SIZE = 4


def clear_operator_cache() -> None:
    """Drop cached operators (and the device memory their plans hold)."""
    with _OP_CACHE_LOCK:
        _OP_CACHE.clear()


def build_sketch(spec: SketchSpec, m: int) -> SketchOperator:
    """Realise ``spec`` for source dimension ``m`` (sketch.py:84-127).

    Operators are immutable and a (spec, m) pair always yields the same one
    bitwise, so the most recent ones are cached: repeated
    solves with the same spec skip the host draws and the device upload."""
    if m < 1:
        raise SpecError(f"source dimension must be >= 1, got {m}")
    key = (spec.kind, spec.embed_dim, spec.seed & ((1 << 64) - 1), spec.sparsity, m)
    with _OP_CACHE_LOCK:
        op = _OP_CACHE.get(key)
        if op is not None:
            _OP_CACHE.move_to_end(key)
            return op
    op = _build_sketch(spec, m)
    if OP_CACHE_SIZE > 0:
        with _OP_CACHE_LOCK:
            _OP_CACHE[key] = op
            while len(_OP_CACHE) > OP_CACHE_SIZE:
                _OP_CACHE.popitem(last=False)
    return op


def _build_sketch(spec: SketchSpec, m: int) -> SketchOperator:
    if spec.kind == "identity":
        return SketchOperator(kind="identity", source_dim=m, target_dim=m)
    d = spec.embed_dim
    if d > m:
        raise SpecError(f"embed_dim {d} exceeds source dimension {m} for kind {spec.kind!r}")
    key = derive_seed(spec.seed, spec.kind, m)
    if spec.kind == "gaussian":
        return SketchOperator("gaussian", m, d, key=key)
    if spec.kind == "countsketch":
        if torch.cuda.is_available():
            # draws on the device (bit-identical to the host walk)
            rows_d = torch.empty(m, dtype=torch.int32, device="cuda")
            signs_d = torch.empty(m, dtype=torch.int8, device="cuda")
            _native.call("skl_rng_countsketch_device", key, m, d, _native.ptr(rows_d),
                         _native.ptr(signs_d), current_stream())
            return SketchOperator("countsketch", m, d, key=key, device_hashes=(rows_d, signs_d))
        rows, signs = _native.rng_countsketch(key, m, d)
        return SketchOperator("countsketch", m, d, rows=_freeze(rows), signs=_freeze(signs),
                              key=key)
    if spec.kind == "sparsesign":
        # sketch.py:104-115: the draws come from numpy's own Generator on the
        # operator stream (bit-identical by construction, including the
        # argpartition and redraw paths); the apply runs on the device
        s = spec.sparsity
        if s > d:
            raise SpecError(f"sparsesign needs sparsity <= embed_dim, got s={s}, d={d}")
        rng = stream(key)
        rows = _sample_distinct_rows(rng, m, d, s)
        signs = 2.0 * rng.integers(0, 2, size=(m, s)) - 1.0
        return SketchOperator("sparsesign", m, d, rows=_freeze(rows.astype(np.int32)),
                              signs=_freeze(signs.astype(np.int8)), key=key, sparsity=s)
    m_pad = 1 << (m - 1).bit_length()
    signs8, sample = _native.rng_srht(key, m_pad, d)
    return SketchOperator("srht", m, d, sign_diag=_freeze(signs8.astype(np.float64)),
                          row_sample=_freeze(sample), padded_dim=m_pad, key=key)


def _sample_distinct_rows(rng, m: int, d: int, s: int) -> np.ndarray:
    """m independent uniform samples of s distinct rows out of d -- the
    reference's draw sequence (sketch.py:130-149) on the same Generator."""
    if s == d:
        return np.tile(np.arange(d, dtype=np.int64), (m, 1))
    if d <= 4 * s * s:
        out = np.empty((m, s), dtype=np.int64)
        chunk = max(1, _SAMPLE_CHUNK_ENTRIES // d)
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            keys = rng.random((hi - lo, d))
            out[lo:hi] = np.argpartition(keys, s - 1, axis=1)[:, :s]
        return out
    rows = rng.integers(0, d, size=(m, s))
    while True:
        srt = np.sort(rows, axis=1)
        bad = np.flatnonzero(np.any(np.diff(srt, axis=1) == 0, axis=1))
        if bad.size == 0:
            return rows
        rows[bad] = rng.integers(0, d, size=(bad.size, s))


# ------------------------------------------------------------------ applies
def _aligned(t, ld: int, cols: int):
    """Return (tensor, ld) satisfying the kernels' 16-byte alignment rules,
    copying on the device when the caller's layout does not."""
    if t.data_ptr() % 16 == 0 and (ld % 2 == 0 or cols == 1):
        return t, ld
    rows = t.shape[0]
    ld2 = (rows + 1) // 2 * 2
    out = device_f64((rows, cols), fortran=True, ld=ld2)
    out.copy_(t)
    return out, ld2


# Column length (bytes) up to which few-column applies take the ordered
# bucket walk: one column's gathers then stay resident in the 126 MB L2.
_ORDERED_MAX_COLUMN_BYTES = 64 << 20


def _few_long_columns(m: int, ncols: int) -> bool:
    """True where the column kernels would split the rows into partitions
    (too few columns to fill the SMs on a long source; csrc/skl_countsketch.cu
    countsketch_owned_launch / countsketch_launch) -- the ordered bucket walk
    keeps those applies bitwise instead."""
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return ncols * 2 < sms and m > (1 << 18) and 8 * m <= _ORDERED_MAX_COLUMN_BYTES


def _countsketch_dense_device(op: SketchOperator, A, lda: int, n: int, b=None):
    """SA (d x n column-major tensor) and Sb (d) or None, all on device."""
    d, m = op.target_dim, op.source_dim
    A, lda = _aligned(A, lda, n)
    if b is not None and b.data_ptr() % 16:
        b = b.clone()
    SA = device_f64((d, n), fortran=True)
    Sb = device_f64((d,)) if b is not None else None
    if _few_long_columns(m, n + (b is not None)):
        brow, bptr, signs = op.device_buckets()
        scale = 1.0 / math.sqrt(op.sparsity) if op.kind == "sparsesign" else 1.0
        _native.call("skl_countsketch_dense_ordered", _native.ptr(A), m, n, lda, _native.ptr(b),
                     _native.ptr(brow), _native.ptr(bptr), _native.ptr(signs), scale, d,
                     _native.ptr(SA), d, _native.ptr(Sb), 0, current_stream())
        return SA, Sb
    op.device_plan().apply(A, m, n, lda, b, SA, d, Sb)
    return SA, Sb


def _countsketch_dense_host(op: SketchOperator, A: np.ndarray, n: int,
                            b: np.ndarray | None = None):
    """Host buffers in, host SA/Sb out; H2D streamed under the kernel."""
    plan = op.device_plan()
    d, m = op.target_dim, op.source_dim
    A = np.asfortranarray(A)
    SA = np.empty((d, n), dtype=np.float64, order="F")
    Sb = np.empty(d, dtype=np.float64) if b is not None else None
    plan.apply_host(A, m, n, A.shape[0] if A.ndim == 2 else m, b, SA, d, Sb)
    return SA, Sb


def _countsketch_csr_device(op: SketchOperator, A: SparseMatrix):
    require_cuda()
    indptr, indices, values = A.device_arrays()
    brow, bptr, signs = op.device_buckets()
    d, n = op.target_dim, A.cols
    SA = device_f64((d, n), fortran=True)
    if op.kind == "sparsesign":
        _native.call("skl_sparsesign_csr", _native.ptr(indptr), _native.ptr(indices),
                     _native.ptr(values), A.rows, n, _native.ptr(brow), _native.ptr(bptr),
                     _native.ptr(signs), 1.0 / math.sqrt(op.sparsity), d, _native.ptr(SA), d,
                     current_stream())
        return SA
    _native.call("skl_countsketch_csr", _native.ptr(indptr), _native.ptr(indices),
                 _native.ptr(values), A.rows, n, _native.ptr(brow), _native.ptr(bptr),
                 _native.ptr(signs), d, _native.ptr(SA), d, current_stream())
    return SA


def _srht_device(op: SketchOperator, A, lda: int, n: int):
    signs, sample = op.device_srht()
    A, lda = _aligned(A, lda, n)
    if lda % 2 and n > 1:
        A, lda = _aligned(A.clone(), lda, n)
    d = op.target_dim
    SA = device_f64((d, n), fortran=True)
    _native.call("skl_srht_dense", _native.ptr(A), op.source_dim, n, lda, _native.ptr(signs),
                 _native.ptr(sample), op.padded_dim, d, _native.ptr(SA), d, current_stream())
    return SA


def _srht_device_ab(op: SketchOperator, A, lda: int, n: int, b):
    """(S A, S b) of a dense [A | b] in one SRHT pass (b as the last column)."""
    signs, sample = op.device_srht()
    A, lda = _aligned(A, lda, n)
    if lda % 2 and n > 1:
        A, lda = _aligned(A.clone(), lda, n)
    d = op.target_dim
    SA = device_f64((d, n), fortran=True)
    Sb = device_f64((d,))
    _native.call("skl_srht_dense_ab", _native.ptr(A), op.source_dim, n, lda, _native.ptr(b),
                 _native.ptr(signs), _native.ptr(sample), op.padded_dim, d, 0, _native.ptr(SA), d,
                 _native.ptr(Sb), 0, current_stream())
    return SA, Sb


def _gaussian_device(op: SketchOperator, A, lda: int, n: int):
    G, ldg = op.device_gaussian()
    A, lda = _aligned(A, lda, n)
    d = op.target_dim
    SA = device_f64((d, n), fortran=True)
    _native.call("skl_gemm_f64", _native.ptr(G), ldg, _native.ptr(A), lda, _native.ptr(SA), d,
                 d, n, op.source_dim, 0, current_stream())
    return SA


def _apply_device(op: SketchOperator, operand):
    """S @ operand on the device.  operand: DenseMatrix | SparseMatrix | Vector.
    Returns a column-major tensor (d x n) or a vector tensor (d)."""
    require_cuda()
    if isinstance(operand, SparseMatrix):
        if op.kind in ("countsketch", "sparsesign"):
            return _countsketch_csr_device(op, operand)
        if op.kind == "identity":
            return to_device(operand.to_scipy().toarray(order="F"))
        # srht / gaussian: the reference densifies the CSR input
        # (sketch.py:205-206, 214) -- do the same on the device.
        dense = to_device(np.asfortranarray(operand.to_scipy().toarray()))
        return _apply_dense_tensor(op, dense, operand.rows, operand.cols)
    if isinstance(operand, Vector):
        v = operand.data if operand.on_device else to_device(operand.data)
        out = _apply_dense_tensor(op, v.reshape(-1, 1), operand.len, 1, lda=operand.len)
        return out.reshape(-1)
    t = operand.data if operand.on_device else to_device(operand.data)
    return _apply_dense_tensor(op, t, operand.rows, operand.cols, lda=operand.ld)


def _apply_dense_tensor(op: SketchOperator, t, m: int, n: int, lda: int | None = None):
    lda = lda if lda is not None else (int(t.stride(1)) if n > 1 else m)
    if op.kind == "identity":
        return t.clone()
    if op.kind in ("countsketch", "sparsesign"):
        SA, _ = _countsketch_dense_device(op, t, lda, n)
        return SA
    if op.kind == "srht":
        return _srht_device(op, t, lda, n)
    if op.kind == "gaussian":
        return _gaussian_device(op, t, lda, n)
    raise SpecError(f"kind {op.kind!r} is not implemented by the B200 engine")


def apply_to_matrix(op: SketchOperator, A: Matrix) -> DenseMatrix:
    """S A as a dense d x n matrix (sketch.py:180-188).  Host carriers give a
    host result, device carriers a device result."""
    if A.rows != op.source_dim:
        raise ShapeError(f"operator expects {op.source_dim} rows, matrix has {A.rows}")
    if isinstance(A, DenseMatrix) and not A.on_device and op.kind == "countsketch":
        SA, _ = _countsketch_dense_host(op, A.data, A.cols)
        return DenseMatrix(SA)
    out = _apply_device(op, A)
    if isinstance(A, DenseMatrix) and A.on_device:
        return DenseMatrix(out)
    return DenseMatrix(out.cpu().numpy())


def apply_to_vector(op: SketchOperator, b: Vector) -> Vector:
    """S b as a length-d vector (sketch.py:191-195)."""
    if b.len != op.source_dim:
        raise ShapeError(f"operator expects length {op.source_dim}, vector has {b.len}")
    out = _apply_device(op, b)
    return Vector(out if b.on_device else out.cpu().numpy())


def fwht_inplace(x):
    """In-place unnormalised FWHT along the leading dimension (sketch.py:152-177),
    computed on the device.  Same argument checks as the reference."""
    a = x if isinstance(x, np.ndarray) else np.asarray(x)
    if a.dtype != np.float64:
        raise ValueError("fwht_inplace requires a float64 array")
    if a.ndim not in (1, 2):
        raise ShapeError("fwht_inplace expects a 1-d or 2-d array")
    n = a.shape[0]
    if n < 1 or (n & (n - 1)) != 0:
        raise ShapeError(f"fwht_inplace requires a power-of-two length, got {n}")
    if not (a.flags.c_contiguous and a.flags.writeable):
        raise ValueError("fwht_inplace requires a writable C-contiguous array")
    cols = 1 if a.ndim == 1 else a.shape[1]
    dev = to_device(np.asfortranarray(a.reshape(n, cols)))
    _native.call("skl_fwht_device", _native.ptr(dev), n, cols, n, current_stream())
    a.reshape(n, cols)[...] = dev.cpu().numpy()
    return x


def materialize(op: SketchOperator) -> DenseMatrix:
    """Explicit d x m matrix equal to the operator (sketch.py:226-242).
    Test/inspection helper, guarded at d*m <= 1e7 entries."""
    d, m = op.target_dim, op.source_dim
    if d * m > _MATERIALIZE_GUARD:
        raise CapacityError(f"materialize guard exceeded: {d}x{m} > {_MATERIALIZE_GUARD} entries")
    if op.kind == "identity":
        return DenseMatrix(np.eye(m))
    if op.kind == "gaussian":
        return DenseMatrix(op.gaussian_entries.copy())
    if op.kind == "countsketch":
        out = np.zeros((d, m))
        out[op.rows, np.arange(m)] = op.signs
        return DenseMatrix(out)
    if op.kind == "sparsesign":
        return DenseMatrix(op.sparse_map.toarray())
    cols = np.arange(m, dtype=np.int64)
    parity = np.bitwise_count(op.row_sample[:, None] & cols[None, :]) & 1
    h_rows = 1.0 - 2.0 * parity.astype(np.float64)
    return DenseMatrix(h_rows * op.sign_diag[:m][None, :] / math.sqrt(d))
