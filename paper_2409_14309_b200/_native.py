"""ctypes binding of the C-ABI in ``include/sketchls_b200.h``.

The shared library ``_lib/libsketchls_b200.so`` is built in-tree by
``_build.py`` (``__graft_entry__.build()``).  There is no fallback: if the
library is missing or a call fails, the mapped exception is raised.
Device buffers are passed as raw pointers (``torch.Tensor.data_ptr()``) and
the caller's current CUDA stream as ``void*``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (
    CapacityError,
    DeviceError,
    ShapeError,
    SingularFactorError,
    SketchlsError,
    SpecError,
)

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsketchls_b200.so"

_lib = None
_lock = threading.Lock()

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_ptr = ctypes.c_void_p
c_dbl_p = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "skl_last_error": (ctypes.c_char_p, []),
    "skl_abi_version": (c_int, []),
    "skl_splitmix64": (c_u64, [c_u64]),
    "skl_rng_u32": (c_int, [c_u64, c_u64, c_i64, c_ptr]),
    "skl_rng_u64": (c_int, [c_u64, c_u64, c_i64, c_ptr]),
    "skl_rng_countsketch": (c_int, [c_u64, c_i64, c_i64, c_ptr, c_ptr, c_int, c_ptr]),
    "skl_rng_srht": (c_int, [c_u64, c_i64, c_i64, c_ptr, c_ptr, c_int]),
    "skl_countsketch_plan": (
        c_int, [c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_int]),
    "skl_sparsesign_plan": (
        c_int, [c_ptr, c_ptr, c_i64, c_int, c_i64, c_i64, c_int, c_ptr, c_ptr, c_int]),
    "skl_sparsesign_dense": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, ctypes.c_double,
         c_ptr, c_i64, c_ptr, c_int, c_int, c_ptr]),
    "skl_countsketch_dense": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr,
         c_i64, c_ptr, c_int, c_int, c_ptr],
    ),
    "skl_countsketch_plan_owned": (
        c_int, [c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_int]),
    "skl_countsketch_dense_owned": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr,
         c_i64, c_ptr, c_int, c_int, c_ptr],
    ),
    "skl_countsketch_dense_host": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr,
         c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    ),
    "skl_rng_countsketch_device": (c_int, [c_u64, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "skl_countsketch_plan_owned_device": (
        c_int, [c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_sparsesign_plan_owned": (
        c_int, [c_ptr, c_ptr, c_i64, c_i64, c_i64, c_i64, c_int, c_ptr, c_ptr, c_int]),
    "skl_sparsesign_dense_owned": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int,
         ctypes.c_double, c_ptr, c_i64, c_ptr, c_int, c_int, c_ptr],
    ),
    "skl_sparsesign_csr": (
        c_int,
        [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, ctypes.c_double, c_i64, c_ptr,
         c_i64, c_ptr],
    ),
    "skl_countsketch_dense_owned_host": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_int, c_ptr,
         c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    ),
    "skl_lsqr_work_size": (c_i64, [c_i64, c_i64]),
    "skl_lsqr_counter_size": (c_i64, [c_i64]),
    "skl_lsqr_gemv_n": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, ctypes.c_double, ctypes.c_double, c_ptr, c_ptr, c_ptr,
         c_ptr, c_ptr, c_ptr],
    ),
    "skl_lsqr_gemv_t": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, ctypes.c_double, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr],
    ),
    "skl_lsqr_trsv_t": (
        c_int, [c_ptr, c_i64, c_i64, c_ptr, ctypes.c_double, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_trsv_n": (c_int, [c_ptr, c_i64, c_i64, ctypes.c_double, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_rinv_blocks": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "skl_lsqr_rinv_full": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "skl_lsqr_step_full_dev": (
        c_int, [c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_state_size": (c_i64, []),
    "skl_lsqr_fused_dev": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_step_dev": (
        c_int,
        [c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_trsv_t_inv": (
        c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr, ctypes.c_double, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_trsv_n_inv": (
        c_int, [c_ptr, c_i64, c_i64, c_ptr, ctypes.c_double, c_ptr, c_ptr, c_ptr]),
    "skl_lsqr_spmv": (
        c_int,
        [c_ptr, c_ptr, c_ptr, c_i64, c_ptr, ctypes.c_double, ctypes.c_double, c_ptr, c_ptr, c_ptr,
         c_ptr, c_ptr, c_ptr],
    ),
    "skl_lsqr_csc_t": (
        c_int,
        [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, ctypes.c_double, c_ptr, c_ptr, c_ptr],
    ),
    "skl_lsqr_xw": (
        c_int, [c_i64, ctypes.c_double, ctypes.c_double, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_srht_dense": (
        c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "skl_srht_dense_ab": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr,
         c_int, c_ptr]),
    "skl_srht_dense_shard": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "skl_fwht_device": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr]),
    "skl_srht_sign_words": (c_i64, [c_i64]),
    "skl_srht_pack_signs": (c_int, [c_ptr, c_i64, c_ptr]),
    "skl_gaussian_set_tables": (c_int, [c_ptr, c_ptr, c_ptr]),
    "skl_rng_gaussian_device": (c_int, [c_u64, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "skl_rng_normal_device": (c_int, [c_u64, c_u64, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr]),
    "skl_rng_gaussian_host": (c_int, [c_u64, c_i64, c_ptr]),
    "skl_gaussian_segment_words": (c_i64, []),
    "skl_gaussian_band_begin": (c_int, [c_u64, c_i64, c_i64, c_ptr, c_ptr, c_ptr]),
    "skl_gaussian_band_count": (c_int, [c_ptr, c_ptr, c_ptr]),
    "skl_gaussian_band_write": (
        c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, ctypes.c_double, c_ptr]),
    "skl_gaussian_band_free": (None, [c_ptr, c_ptr]),
    "skl_gemm_f64": (
        c_int, [c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_i64, c_i64, c_i64, c_i64, c_int, c_ptr]),
    "skl_countsketch_buckets": (c_int, [c_ptr, c_i64, c_i64, c_ptr, c_ptr]),
    "skl_countsketch_csr": (
        c_int,
        [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr],
    ),
    "skl_countsketch_dense_ordered": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, ctypes.c_double, c_i64, c_ptr,
         c_i64, c_ptr, c_int, c_ptr],
    ),
    "skl_lsqr_fused_work_size": (c_i64, [c_i64]),
    "skl_lsqr_fused": (
        c_int,
        [c_ptr, c_i64, c_i64, c_i64, c_ptr, ctypes.c_double, ctypes.c_double, c_ptr, ctypes.c_double,
         c_ptr, c_ptr,
         c_ptr, c_ptr, c_ptr, c_ptr],
    ),
    "skl_qr_solve": (
        c_int,
        [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr,
         c_ptr],
    ),
    "skl_qr_solve_async": (
        c_int,
        [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr,
         c_ptr],
    ),
    "skl_cqr_supported": (c_int, [c_i64, c_i64]),
    "skl_cqr_solve_async": (c_int, [c_ptr, c_i64, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_residual_dense": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_residual_dense_async": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_residual_csr_async": (c_int, [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "skl_sum_slots": (c_int, [c_ptr, c_i64, c_i64, c_i64, c_i64, c_i64, c_ptr, c_i64, c_ptr]),
    "skl_reduce_peers": (c_int, [c_ptr, c_int, c_i64, c_i64, c_ptr, c_ptr]),
    "skl_residual_csr": (c_int, [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
}

_STATUS = {
    1: ShapeError,
    2: SpecError,
    3: SingularFactorError,
    4: CapacityError,
    5: DeviceError,
    6: ValueError,
    7: DeviceError,
}


_tables_installed = False


def install_gaussian_tables() -> None:
    """Hand numpy's ziggurat tables (read from the installed library) to the
    native generator once per process."""
    global _tables_installed
    if _tables_installed:
        return
    from ._ziggurat import tables

    ki, wi, fi = tables()
    call("skl_gaussian_set_tables", ptr(ki), ptr(wi), ptr(fi))
    _tables_installed = True


def rng_gaussian_host(key: int, count: int) -> np.ndarray:
    """First `count` standard normals of Generator(Philox(key)) (host, libm)."""
    install_gaussian_tables()
    out = np.empty(count, dtype=np.float64)
    call("skl_rng_gaussian_host", key, count, ptr(out))
    return out


def _ensure_built() -> None:
    """Build the library when it is missing or older than any of its sources
    (a stale build would silently run old kernels).  A file lock keeps
    concurrent processes (torchrun ranks) from building at the same time."""
    import fcntl

    from . import _build

    if LIB_PATH.exists() and not _build._stale():
        return
    LIB_PATH.parent.mkdir(exist_ok=True)
    with open(LIB_PATH.parent / ".build.lock", "w") as fh:
        fcntl.flock(fh, fcntl.LOCK_EX)
        try:
            if not LIB_PATH.exists() or _build._stale():
                _build.build()
        finally:
            fcntl.flock(fh, fcntl.LOCK_UN)


def lib() -> ctypes.CDLL:
    """The loaded library (built on first use if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            _ensure_built()
            if not LIB_PATH.exists():
                raise DeviceError(f"native library missing: {LIB_PATH}")
            handle = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().skl_last_error().decode("utf-8", "replace")
    raise _STATUS.get(status, SketchlsError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr_array(addrs) -> ctypes.Array:
    """Host array of device addresses (e.g. the ranks' symmetric buffers)."""
    return (ctypes.c_void_p * len(addrs))(*[int(a) for a in addrs])


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, int):  # already a device address (e.g. a peer buffer)
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


# ----------------------------------------------------------------- host RNG
def rng_u32(key: int, offset: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint32)
    call("skl_rng_u32", key, offset, count, ptr(out))
    return out


def rng_u64(key: int, offset: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    call("skl_rng_u64", key, offset, count, ptr(out))
    return out


def rng_countsketch(key: int, m: int, d: int, threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    rows = np.empty(m, dtype=np.int32)
    signs = np.empty(m, dtype=np.int8)
    call("skl_rng_countsketch", key, m, d, ptr(rows), ptr(signs), threads, None)
    return rows, signs


def rng_srht(key: int, m_pad: int, d: int, threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    signs = np.empty(m_pad, dtype=np.int8)
    sample = np.empty(d, dtype=np.int64)
    call("skl_rng_srht", key, m_pad, d, ptr(signs), ptr(sample), threads)
    return signs, sample


# Register-owned plans cover d <= 16 warps x 32 lanes x 8 slots; larger
# embeddings use lane lists (shared-memory bucket sums).
OWNED_MAX_D = 4096
OWNED_CHUNK = 8184   # rows per chunk (<= 8184: 13-bit row field incl. the zero slot)
OWNED_SMALL_CHUNK = 4096  # short sources (<= 4 full chunks)
LANES_CHUNK = 2048


def plan_geometry(d: int, kind: str | None = None, m: int | None = None) -> tuple[str, int, int]:
    """(plan kind, chunk rows, consumer warps) of the CountSketch plan for
    embed_dim d: "owned" (register-owned buckets, 4 or 8 per thread) when
    d <= 4096, else
    "lanes" (shared-memory accumulators, lane lists).  ``kind`` forces one
    (tests exercise both kernels on the same operator).  Short sources (m
    rows, at most four full chunks) get half-size chunks: the kernel's ring
    then needs half the shared memory, two or three column CTAs share an SM
    and the whole grid runs in one wave."""
    kind = kind or ("owned" if d <= OWNED_MAX_D else "lanes")
    if kind == "owned":
        if d > OWNED_MAX_D:
            raise ValueError(f"owned plan needs d <= {OWNED_MAX_D}, got {d}")
        warps = 8 if d <= 1024 else 16
        if d <= 2048:  # 4 slots per thread: 13-bit row field
            chunk = OWNED_CHUNK if m is None or m > 4 * OWNED_CHUNK else OWNED_SMALL_CHUNK
            forced = int(os.environ.get("SKL_OWNED_CHUNK", "0") or 0)  # A/B knob
            if forced >= 8:
                chunk = min(OWNED_CHUNK, forced // 8 * 8)
        else:  # 8 slots: 12-bit row field
            chunk = 4088
        return "owned", chunk, warps
    if kind != "lanes":
        raise ValueError(f"unknown plan kind {kind!r}")
    return "lanes", LANES_CHUNK, (16 if d >= 1024 else 8)


def countsketch_plan(rows: np.ndarray, signs: np.ndarray, d: int, chunk: int, warps: int,
                     threads: int = 0, spr: int = 1) -> tuple[np.ndarray, np.ndarray, int]:
    """(lanes u32, chunk_off i64 [nch+1], max block words) -- see the header;
    ``spr`` entries per source row (a sparse sign plan, rows/signs flattened)."""
    m = rows.shape[0] // spr
    nch = (m + chunk - 1) // chunk
    off = np.zeros(nch + 1, dtype=np.int64)
    if spr == 1:
        fn, pre = "skl_countsketch_plan", (ptr(rows), ptr(signs), m, d, chunk, warps)
    else:
        fn, pre = "skl_sparsesign_plan", (ptr(rows), ptr(signs), m, spr, d, chunk, warps)
    call(fn, *pre, None, ptr(off), threads)
    lanes = np.empty(int(off[-1]), dtype=np.uint32)
    call(fn, *pre, ptr(lanes), ptr(off), threads)
    return lanes, off, int(np.diff(off).max())


def countsketch_plan_owned(rows: np.ndarray, signs: np.ndarray, d: int, chunk: int, warps: int,
                           threads: int = 0, spr: int = 1) -> tuple[np.ndarray, np.ndarray, int]:
    """(lanes u16, chunk_off i64 [nch+1], max block words) of the register-owned
    plan; ``spr`` entries per source row (rows/signs flattened m x spr)."""
    m = rows.shape[0] // spr
    nch = (m + chunk - 1) // chunk
    off = np.zeros(nch + 1, dtype=np.int64)
    if spr == 1:
        args = lambda lanes: (ptr(rows), ptr(signs), m, d, chunk, warps, lanes, ptr(off), threads)  # noqa: E731
        fn = "skl_countsketch_plan_owned"
    else:
        args = lambda lanes: (ptr(rows), ptr(signs), m, spr, d, chunk, warps, lanes, ptr(off),  # noqa: E731
                              threads)
        fn = "skl_sparsesign_plan_owned"
    call(fn, *args(None))
    lanes = np.empty(int(off[-1]), dtype=np.uint16)
    call(fn, *args(ptr(lanes)))
    return lanes, off, int(np.diff(off).max())


def countsketch_buckets(rows: np.ndarray, d: int) -> tuple[np.ndarray, np.ndarray]:
    m = rows.shape[0]
    brow = np.empty(m, dtype=np.int32)
    bptr = np.empty(d + 1, dtype=np.int64)
    call("skl_countsketch_buckets", ptr(rows), m, d, ptr(brow), ptr(bptr))
    return brow, bptr


def srht_pack_signs(signs: np.ndarray) -> np.ndarray:
    """Packed sign words of an SRHT sign diagonal (int8 +-1, length m_pad)."""
    m_pad = signs.shape[0]
    B = min(m_pad, 4096)
    words = int(lib().skl_srht_sign_words(B)) * (m_pad // B)
    out = np.zeros(max(words, 8), dtype=np.uint16)
    call("skl_srht_pack_signs", ptr(np.ascontiguousarray(signs, dtype=np.int8)), m_pad, ptr(out))
    return out
