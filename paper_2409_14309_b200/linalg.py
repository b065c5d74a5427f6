"""Carriers and the device reduced-solve kernels.

Carriers keep the reference's conventions
(/root/reference/pkg/src/sketchls/linalg.py:31-133): dense matrices are
fp64 column-major, sparse matrices are CSR with int64 indices and strictly
increasing columns, every carrier is immutable after construction.  A
carrier may additionally hold a CUDA tensor (device-resident data, the
engine's native habitat); host numpy data is moved to the device by the
kernels that consume it.

``economy_qr`` (linalg.py:166-192) and the inverse-R solve
(linalg.py:214-218) run on the device through ``skl_qr_solve``.
"""

from __future__ import annotations

import math
import os
import threading

from dataclasses import dataclass

import numpy as np
import scipy.sparse

from . import _native
from ._device import current_stream, device_f64, require_cuda, to_device, torch
from .errors import ShapeError, SingularFactorError

# Relative threshold below which a diagonal entry of R marks the input as
# rank deficient (linalg.py:23).
RANK_TOL = 1e-14


def _freeze(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


def _is_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


@dataclass(frozen=True)
class DenseMatrix:
    """Column-major float64 matrix with at least one row and column.

    ``data`` is a read-only Fortran-ordered numpy array (host) or a CUDA
    float64 tensor with column-major strides (device)."""

    data: object

    def __post_init__(self) -> None:
        if _is_tensor(self.data):
            t = self.data
            if t.dtype != torch.float64 or not t.is_cuda:
                raise ValueError("device dense matrix must be a CUDA float64 tensor")
            if t.dim() != 2:
                raise ShapeError(f"dense matrix must be 2-d, got ndim={t.dim()}")
            if t.shape[0] < 1 or t.shape[1] < 1:
                raise ShapeError(f"dense matrix must be nonempty, got shape {tuple(t.shape)}")
            if not (t.stride(0) == 1 and (t.shape[1] == 1 or t.stride(1) >= t.shape[0])):
                t = t.t().contiguous().t()
            if not bool(torch.isfinite(t).all()):
                raise ValueError("dense matrix entries must be finite")
            object.__setattr__(self, "data", t)
            return
        a = np.asfortranarray(self.data, dtype=np.float64)
        if a.ndim != 2:
            raise ShapeError(f"dense matrix must be 2-d, got ndim={a.ndim}")
        if a.shape[0] < 1 or a.shape[1] < 1:
            raise ShapeError(f"dense matrix must be nonempty, got shape {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("dense matrix entries must be finite")
        object.__setattr__(self, "data", _freeze(a))

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def cols(self) -> int:
        return int(self.data.shape[1])

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.data)

    @property
    def ld(self) -> int:
        if self.on_device:
            return int(self.data.stride(1)) if self.cols > 1 else self.rows
        return self.rows

    def to_numpy(self) -> np.ndarray:
        if self.on_device:
            return np.asfortranarray(self.data.cpu().numpy())
        return self.data


@dataclass(frozen=True)
class SparseMatrix:
    """Compressed-row float64 matrix with strictly increasing column indices
    per row (linalg.py:56-114).  Host arrays; a device copy is cached on
    first use by the kernels."""

    rows: int
    cols: int
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        if self.rows < 1 or self.cols < 1:
            raise ShapeError(f"sparse matrix must be nonempty, got {self.rows}x{self.cols}")
        indptr = np.ascontiguousarray(self.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(self.indices, dtype=np.int64)
        values = np.ascontiguousarray(self.values, dtype=np.float64)
        if indptr.ndim != 1 or indptr.shape[0] != self.rows + 1:
            raise ShapeError("row pointers must have length rows+1")
        if indptr[0] != 0 or np.any(np.diff(indptr) < 0):
            raise ValueError("row pointers must start at 0 and be nondecreasing")
        nnz = int(indptr[-1])
        if indices.shape[0] != nnz or values.shape[0] != nnz:
            raise ShapeError("index/value arrays must match the final row pointer")
        if nnz and (indices.min() < 0 or indices.max() >= self.cols):
            raise ValueError("column indices out of range")
        if nnz > 1:
            diffs = np.diff(indices)
            row_starts = np.zeros(nnz - 1, dtype=bool)
            interior = indptr[1:-1]
            interior = interior[(interior > 0) & (interior < nnz)]
            row_starts[interior - 1] = True
            if np.any((diffs <= 0) & ~row_starts):
                raise ValueError("column indices must be strictly increasing within each row")
        if not np.all(np.isfinite(values)):
            raise ValueError("sparse matrix values must be finite")
        object.__setattr__(self, "indptr", _freeze(indptr))
        object.__setattr__(self, "indices", _freeze(indices))
        object.__setattr__(self, "values", _freeze(values))
        object.__setattr__(self, "_dev", {})

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix(
            (self.values, self.indices, self.indptr), shape=(self.rows, self.cols)
        )

    @classmethod
    def from_scipy(cls, mat) -> "SparseMatrix":
        csr = scipy.sparse.csr_matrix(mat)
        csr.sort_indices()
        csr.sum_duplicates()
        return cls(csr.shape[0], csr.shape[1], csr.indptr, csr.indices, csr.data)

    def densify(self) -> DenseMatrix:
        return DenseMatrix(self.to_scipy().toarray())

    def device_arrays(self):
        """(indptr, indices, values) as CUDA tensors, uploaded once."""
        require_cuda()
        dev = torch.cuda.current_device()
        cache = self._dev
        if dev not in cache:
            cache[dev] = (to_device(self.indptr), to_device(self.indices),
                          to_device(self.values))
        return cache[dev]

    def device_csc(self):
        """(colptr int64 cols+1, rowidx int32, values) of the same matrix in
        compressed-column form on the current device, built once from the
        device CSR arrays (a stable sort of the nonzeros by column, so the
        rows of every column stay ascending -- the order scipy's folds use)
        and kept with the operand, like the device copy itself (LSQR's
        A^T u; round 1 rebuilt it for every solve)."""
        require_cuda()
        key = ("csc", torch.cuda.current_device())
        cache = self._dev
        if key not in cache:
            indptr, indices, values = self.device_arrays()
            counts = indptr[1:] - indptr[:-1]
            rows = torch.repeat_interleave(
                torch.arange(self.rows, dtype=torch.int32, device=indptr.device), counts)
            order = torch.sort(indices, stable=True).indices
            colptr = torch.zeros(self.cols + 1, dtype=torch.int64, device=indptr.device)
            colptr[1:] = torch.cumsum(torch.bincount(indices, minlength=self.cols), 0)
            cache[key] = (colptr, rows[order].contiguous(), values[order].contiguous())
        return cache[key]


@dataclass(frozen=True)
class Vector:
    """Contiguous float64 vector (linalg.py:117-133); host numpy or CUDA tensor."""

    data: object

    def __post_init__(self) -> None:
        if _is_tensor(self.data):
            t = self.data
            if t.dtype != torch.float64 or not t.is_cuda:
                raise ValueError("device vector must be a CUDA float64 tensor")
            if t.dim() != 1:
                raise ShapeError(f"vector must be 1-d, got ndim={t.dim()}")
            t = t.contiguous()
            if not bool(torch.isfinite(t).all()):
                raise ValueError("vector entries must be finite")
            object.__setattr__(self, "data", t)
            return
        a = np.ascontiguousarray(self.data, dtype=np.float64)
        if a.ndim != 1:
            raise ShapeError(f"vector must be 1-d, got ndim={a.ndim}")
        if not np.all(np.isfinite(a)):
            raise ValueError("vector entries must be finite")
        object.__setattr__(self, "data", _freeze(a))

    @classmethod
    def _of_solution(cls, x, residual_norm: float) -> "Vector":
        """Wrap a solver's x without the finiteness pass when ||A x - b|| is
        finite (a non-finite entry of x makes the residual non-finite: every
        column of A has a nonzero, or the sketched QR would have stopped),
        sparing a device reduction and a synchronisation per solve; a
        non-finite residual goes through the full check (and its error)."""
        if not math.isfinite(residual_norm):
            return cls(x)
        if _is_tensor(x):
            if x.dtype != torch.float64 or x.dim() != 1 or not x.is_cuda:
                return cls(x)
            v = object.__new__(cls)
            object.__setattr__(v, "data", x.contiguous())
            return v
        return cls(x)

    @property
    def len(self) -> int:
        return int(self.data.shape[0])

    @property
    def on_device(self) -> bool:
        return _is_tensor(self.data)

    def to_numpy(self) -> np.ndarray:
        return self.data.cpu().numpy() if self.on_device else self.data


@dataclass(frozen=True)
class QRFactors:
    """Economy QR factors: Q has orthonormal columns, R is upper triangular
    with nonnegative diagonal (linalg.py:136-142)."""

    Q: DenseMatrix
    R: DenseMatrix


Matrix = DenseMatrix | SparseMatrix


def _as_device_matrix(M: DenseMatrix):
    """(tensor, ld) of M on the current CUDA device (column-major)."""
    if M.on_device:
        return M.data, M.ld
    return to_device(M.data), M.rows


def qr_solve_device(SA, ldsa: int, Sb, d: int, n: int, want_q: bool = False,
                    want_r: bool = False):
    """Device Householder QR + back substitution.  SA: column-major tensor
    (d x n, ld ldsa); Sb: tensor (d) or None.  Returns (x, R, Q) tensors
    (R, Q None unless requested).  Raises SingularFactorError with the
    reference's message (linalg.py:186-191)."""
    x = device_f64((n,))
    R = device_f64((n, n), fortran=True) if want_r else None
    Q = device_f64((d, n), fortran=True) if want_q else None
    bad_col = np.zeros(1, dtype=np.int64)
    bad_val = np.zeros(1, dtype=np.float64)
    _native.call(
        "skl_qr_solve", _native.ptr(SA), ldsa, _native.ptr(Sb), d, n, _native.ptr(x),
        _native.ptr(R), n, _native.ptr(Q), d, _native.ptr(bad_col), _native.ptr(bad_val),
        current_stream())
    return x, R, Q


_RANK_FLAGS = threading.local()


_CQR_OFF = os.environ.get("SKL_QR_HOUSEHOLDER", "") not in ("", "0")


def cholqr_enabled(d: int, n: int) -> bool:
    """Whether the reduced solve of a d x n sketched system takes the
    Cholesky-based path (skl_cqr_solve_async): n + 1 <= 1056 < d, unless
    SKL_QR_HOUSEHOLDER=1 forces the Householder factorisation (A/B knob,
    read at import)."""
    return not _CQR_OFF and bool(_native.lib().skl_cqr_supported(d, n))


def qr_solve_device_async(SA, ldsa: int, Sb, d: int, n: int, flags=None):
    """The reduced solve x = R^{-1} Q^T Sb without its synchronisation:
    returns (x, check) where check() -- to be called once the stream has
    been synchronised (e.g. by the residual pass) -- returns None when x is
    valid, or a replacement x, or raises the SingularFactorError
    skl_qr_solve would have.  Sketched systems with n + 1 <= 1056 < d go
    through the Cholesky-based kernels (csrc/skl_cholqr.cu: a semi-normal
    solve for a well-conditioned SA, shifted CholeskyQR2 otherwise, picked
    on the device); when a Cholesky pivot breaks down, the refinement does
    not contract or the rank check fires, check() re-solves
    with the Householder factorisation, which decides (and words the error
    exactly as linalg.py:186-191).  The flags land in a pinned per-thread
    buffer."""
    if flags is None:  # batched callers pass their own pinned pair per solve
        flags = getattr(_RANK_FLAGS, "buf", None)
        if flags is None:
            flags = torch.empty(2, dtype=torch.float64, pin_memory=True)
            _RANK_FLAGS.buf = flags
    flags_i = flags.view(torch.int64)
    x = device_f64((n,))
    base = flags.data_ptr()
    chol = Sb is not None and cholqr_enabled(d, n)
    if chol:
        _native.call("skl_cqr_solve_async", _native.ptr(SA), ldsa, _native.ptr(Sb), d, n,
                     _native.ptr(x), base, base + 8, current_stream())
    else:
        _native.call(
            "skl_qr_solve_async", _native.ptr(SA), ldsa, _native.ptr(Sb), d, n, _native.ptr(x),
            None, n, None, d, base, base + 8, current_stream())

    def check():
        bad = int(flags_i[0])
        if chol and bad != -1:
            return qr_solve_device(SA, ldsa, Sb, d, n)[0]
        if bad >= 0:
            val = float(flags[1])
            raise SingularFactorError(
                f"input is numerically rank deficient at column {bad} "
                f"(|R[{bad},{bad}]| = {val:.3e})")
        return None

    return x, check


def reduced_solve_device(SA, ldsa: int, Sb, d: int, n: int):
    """x of the sketched system through the path sketch_and_apply takes
    (CholeskyQR2 when eligible, else Householder), synchronised."""
    x, check = qr_solve_device_async(SA, ldsa, Sb, d, n)
    torch.cuda.current_stream().synchronize()
    x2 = check()
    return x if x2 is None else x2


def economy_qr(M: DenseMatrix) -> QRFactors:
    """Householder QR of a tall matrix on the device, M = Q R, diag(R) >= 0
    (linalg.py:166-192).  Factors come back on the side M lives on."""
    if M.rows < M.cols:
        raise ShapeError(f"economy_qr requires rows >= cols, got {M.rows}x{M.cols}")
    require_cuda()
    t, ld = _as_device_matrix(M)
    _, R, Q = qr_solve_device(t, ld, None, M.rows, M.cols, want_q=True, want_r=True)
    if M.on_device:
        return QRFactors(Q=DenseMatrix(Q), R=DenseMatrix(R))
    return QRFactors(Q=DenseMatrix(Q.cpu().numpy()), R=DenseMatrix(R.cpu().numpy()))


def _check_diagonal(r: np.ndarray) -> None:
    zero = np.flatnonzero(np.diagonal(r) == 0.0)
    if zero.size:
        raise SingularFactorError(f"zero diagonal entry at index {int(zero[0])}")


# ---------------------------------------------------------------------------
# Products, triangular solves and the direct solve (linalg.py:148-246), on
# the device through the LSQR kernels (csrc/skl_lsqr.cu) and skl_qr_solve.
# Results live where the operand lives: device tensors for device carriers,
# host arrays otherwise.


def _vec_dev(v: Vector):
    return v.data if v.on_device else to_device(v.data)


def _result(t, on_device: bool) -> Vector:
    return Vector(t if on_device else t.cpu().numpy())


def _operator(A):
    from .solvers import _operator_device

    return _operator_device(A)[0]


def matvec(A, x: Vector) -> Vector:
    """A @ x (linalg.py:148-154); O(nnz) for sparse A."""
    from ._lsqr import _Workspace

    if x.len != A.cols:
        raise ShapeError(f"matvec: A is {A.rows}x{A.cols} but x has length {x.len}")
    require_cuda()
    op = _operator(A)
    out = device_f64((A.rows,))
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    op.mv(_vec_dev(x).contiguous(), 1.0, 0.0, None, out, nrm, _Workspace(A.rows, A.cols),
          current_stream())
    return _result(out, isinstance(A, DenseMatrix) and A.on_device)


def matvec_transpose(A, y: Vector) -> Vector:
    """A.T @ y (linalg.py:157-163); O(nnz) for sparse A."""
    from ._lsqr import _Workspace

    if y.len != A.rows:
        raise ShapeError(f"matvec_transpose: A is {A.rows}x{A.cols} but y has length {y.len}")
    require_cuda()
    op = _operator(A)
    z = device_f64((A.cols,))
    scratch = device_f64((A.rows,))
    op.rmv(_vec_dev(y).contiguous(), 1.0, scratch, z, _Workspace(A.rows, A.cols),
           current_stream())
    return _result(z, isinstance(A, DenseMatrix) and A.on_device)


def solve_triangular(R: DenseMatrix, y: Vector, transposed: bool = False) -> Vector:
    """Solve R z = y (or R^T z = y) for upper-triangular R (linalg.py:195-204)."""
    if R.rows != R.cols:
        raise ShapeError(f"triangular factor must be square, got {R.rows}x{R.cols}")
    if y.len != R.rows:
        raise ShapeError(f"solve_triangular: R is {R.rows}x{R.cols} but y has length {y.len}")
    require_cuda()
    n = R.rows
    Rt, ldr = _as_device_matrix(R)
    diag = torch.diagonal(Rt[:n, :n])
    zero = torch.nonzero(diag == 0.0)
    if zero.numel():
        raise SingularFactorError(f"zero diagonal entry at index {int(zero[0, 0])}")
    yd = _vec_dev(y).contiguous()
    z = device_f64((n,))
    if transposed:
        zeros = torch.zeros(n, dtype=torch.float64, device="cuda")
        nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
        _native.call("skl_lsqr_trsv_t", _native.ptr(Rt), ldr, n, _native.ptr(yd), 0.0,
                     _native.ptr(zeros), _native.ptr(z), _native.ptr(nrm), current_stream())
    else:
        _native.call("skl_lsqr_trsv_n", _native.ptr(Rt), ldr, n, 0.0, _native.ptr(yd),
                     _native.ptr(z), current_stream())
    return _result(z, R.on_device)


def normal_equations_oracle(A: DenseMatrix, b: Vector) -> Vector:
    """argmin ||A x - b|| by Householder QR of A itself, x = R^-1 Q^T b
    (linalg.py:221-232), on the device."""
    if b.len != A.rows:
        raise ShapeError(f"A is {A.rows}x{A.cols} but b has length {b.len}")
    if A.rows < A.cols:
        raise ShapeError(f"need rows >= cols, got {A.rows}x{A.cols}")
    require_cuda()
    t, ld = _as_device_matrix(A)
    x, _, _ = qr_solve_device(t, ld, _vec_dev(b).contiguous(), A.rows, A.cols)
    return _result(x, A.on_device)


def spectral_condition_number(M: DenseMatrix) -> float:
    """sigma_max / sigma_min from all singular values (linalg.py:235-247;
    cuSOLVER through torch); inf when sigma_min is zero."""
    if M.rows < M.cols:
        raise ShapeError(f"need rows >= cols, got {M.rows}x{M.cols}")
    require_cuda()
    t, _ = _as_device_matrix(M)
    s = torch.linalg.svdvals(t[:M.rows, :M.cols])
    smin = float(s[-1])
    return float("inf") if smin == 0.0 else float(s[0]) / smin
