"""CPU ORACLE (test infrastructure only): ctypes access to the plain-C
restatement in oracle/c/philox_oracle.c (random streams) and
oracle/c/apply_oracle.c (column-threaded CountSketch / SRHT applies for the
full-size parity checks), built by oracle/Makefile into
oracle/_build/liboracle.so."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        srcs = [HERE / "c" / "philox_oracle.c", HERE / "c" / "apply_oracle.c", HERE / "Makefile"]
        if not LIB.exists() or LIB.stat().st_mtime < max(p.stat().st_mtime for p in srcs):
            build()
        L = ctypes.CDLL(str(LIB))
        P, I64, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        L.orc_u32.argtypes = [U64, I64, P]
        L.orc_countsketch.argtypes = [U64, I64, I64, P, P]
        L.orc_srht.argtypes = [U64, I64, I64, P, P]
        L.orc_gaussian.argtypes = [U64, I64, P, P, P, ctypes.c_double, ctypes.c_double, P]
        L.orc_countsketch_fold.argtypes = [P, P, I64, I64, P, I64, I64, P]
        L.orc_countsketch_fold_mt.argtypes = [P, P, I64, I64, P, I64, I64, P, I64, ctypes.c_int]
        L.orc_srht_apply.argtypes = [P, I64, I64, I64, P, P, I64, I64, P, I64, ctypes.c_int]
        _lib = L
    return _lib


def u32(key: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint32)
    lib().orc_u32(key, count, out.ctypes.data)
    return out


def countsketch(key: int, m: int, d: int):
    rows = np.empty(m, np.int64)
    signs = np.empty(m, np.float64)
    if lib().orc_countsketch(key, m, d, rows.ctypes.data, signs.ctypes.data):
        raise ValueError("d out of range")
    return rows, signs


def srht(key: int, m_pad: int, d: int):
    signs = np.empty(m_pad, np.float64)
    sample = np.empty(d, np.int64)
    lib().orc_srht(key, m_pad, d, signs.ctypes.data, sample.ctypes.data)
    return signs, sample


def gaussian(key: int, count: int, ki, wi, fi, r: float, inv_r: float) -> np.ndarray:
    out = np.empty(count, np.float64)
    ki = np.ascontiguousarray(ki, np.uint64)
    wi = np.ascontiguousarray(wi, np.float64)
    fi = np.ascontiguousarray(fi, np.float64)
    lib().orc_gaussian(key, count, ki.ctypes.data, wi.ctypes.data, fi.ctypes.data, r, inv_r,
                       out.ctypes.data)
    return out


def countsketch_fold(rows, signs, d: int, A: np.ndarray) -> np.ndarray:
    A = np.asfortranarray(A.reshape(A.shape[0], -1), dtype=np.float64)
    m, n = A.shape
    out = np.empty((d, n), order="F")
    rows = np.ascontiguousarray(rows, np.int64)
    signs = np.ascontiguousarray(signs, np.float64)
    lib().orc_countsketch_fold(rows.ctypes.data, signs.ctypes.data, m, n, A.ctypes.data, m, d,
                               out.ctypes.data)
    return out


def _threads(threads: int | None) -> int:
    import os

    if threads:
        return threads
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def countsketch_apply_mt(rows, signs, d: int, A: np.ndarray, threads: int | None = None):
    """sketch.py:209,212 (`sparse_map @ A`, scipy's csr_matvecs fold) for an
    F-ordered (or 1-d) A, columns spread over host threads; bitwise equal to
    oracle.countsketch_apply.  Returns d x n F-ordered (or d for 1-d A)."""
    vec = A.ndim == 1
    A2 = A.reshape(-1, 1) if vec else A
    if not A2.flags.f_contiguous:
        A2 = np.asfortranarray(A2)
    m, n = A2.shape
    lda = m if n == 1 else A2.strides[1] // 8
    out = np.empty((d, n), order="F")
    rows = np.ascontiguousarray(rows, np.int64)
    signs = np.ascontiguousarray(signs, np.float64)
    if lib().orc_countsketch_fold_mt(rows.ctypes.data, signs.ctypes.data, m, n, A2.ctypes.data,
                                     lda, d, out.ctypes.data, d, _threads(threads)):
        raise RuntimeError("orc_countsketch_fold_mt failed")
    return out[:, 0].copy() if vec else out


def srht_apply_mt(sign_diag, row_sample, m_pad: int, d: int, A: np.ndarray,
                  threads: int | None = None):
    """sketch.py:213-223 (pad, sign, fwht_inplace, sample / sqrt(d)) for an
    F-ordered (or 1-d) A, columns spread over host threads; bitwise equal to
    oracle.srht_apply.  Returns d x n F-ordered (or d for 1-d A)."""
    vec = A.ndim == 1
    A2 = A.reshape(-1, 1) if vec else A
    if not A2.flags.f_contiguous:
        A2 = np.asfortranarray(A2)
    m, n = A2.shape
    lda = m if n == 1 else A2.strides[1] // 8
    out = np.empty((d, n), order="F")
    sg = np.ascontiguousarray(sign_diag, np.float64)
    rs = np.ascontiguousarray(row_sample, np.int64)
    if lib().orc_srht_apply(A2.ctypes.data, m, n, lda, sg.ctypes.data, rs.ctypes.data, m_pad, d,
                            out.ctypes.data, d, _threads(threads)):
        raise RuntimeError("orc_srht_apply failed")
    return out[:, 0].copy() if vec else out
