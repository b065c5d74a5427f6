"""Sketch-and-apply least squares on the B200 engine.

Mirrors /root/reference/pkg/src/sketchls/solvers.py: `LeastSquaresProblem`
:43-60, `SolverOptions` :63-87, `SolveResult` :90-99, `_operator_spec`
:273-279, `_sketch_qr` :282-293, `sketch_and_apply` :296-320 and the
dispatcher `solve` :364-398.  The SAA path keeps everything on the device:
operator build (device RNG, cached plan) -> one sketch pass over [A | b] ->
Householder QR + back substitution -> a second pass for ||Ax - b||.

Sketch-and-precondition (:323-361), LSQR (:110-255, optionally with a
user preconditioner and a per-iteration callback) and the "direct" QR of A
itself (:381-396) run on the device too (_lsqr.py, csrc/skl_lsqr.cu,
skl_qr_solve) for dense and CSR operands.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from ._device import current_stream, device_f64, require_cuda, to_device, torch
from .errors import ShapeError, SingularFactorError, SpecError
from .linalg import (DenseMatrix, Matrix, SparseMatrix, Vector, qr_solve_device,
                     qr_solve_device_async)
from .rng import derive_seed
from .sketch import (
    DEFAULT_KIND,
    SketchSpec,
    _apply_dense_tensor,
    _countsketch_csr_device,
    _countsketch_dense_device,
    _few_long_columns,
    _srht_device_ab,
    build_sketch,
    default_embed_dim,
)

METHODS = ("lsqr", "saa", "sap", "direct")
ENGINE_METHODS = ("saa", "sap", "lsqr", "direct")


@dataclass(frozen=True)
class LeastSquaresProblem:
    """min_x ||A x - b|| (solvers.py:43-60)."""

    A: Matrix
    b: Vector
    x_star: Vector | None = None
    beta: float | None = None

    def __post_init__(self) -> None:
        if self.b.len != self.A.rows:
            raise ShapeError(f"A is {self.A.rows}x{self.A.cols} but b has length {self.b.len}")
        if self.x_star is not None and self.x_star.len != self.A.cols:
            raise ShapeError(f"x_star has length {self.x_star.len}, expected {self.A.cols}")
        if self.beta is not None and not (self.beta >= 0 and math.isfinite(self.beta)):
            raise SpecError(f"beta must be finite and >= 0, got {self.beta}")


@dataclass(frozen=True)
class SolverOptions:
    """Tolerances and sizing knobs (solvers.py:63-87).  Sketch-and-apply uses
    d_factor and the engine's ``devices`` list."""

    atol: float = 1e-10
    btol: float = 1e-10
    max_iter: int | None = None
    d_factor: float = 4.0
    warm_start: bool = True
    # Engine option (not in the reference): CUDA devices the sketch-and-apply
    # shards A's rows over (multidevice.py); None = the current device.
    devices: tuple[int, ...] | None = None

    def __post_init__(self) -> None:
        if not (self.atol > 0 and self.btol > 0):
            raise SpecError("tolerances must be positive")
        if self.max_iter is not None and self.max_iter < 1:
            raise SpecError("max_iter must be >= 1")
        if self.d_factor < 1:
            raise SpecError("d_factor must be >= 1")
        if self.devices is not None:
            from .multidevice import check_devices

            object.__setattr__(self, "devices", check_devices(self.devices))

    def resolve_max_iter(self, n: int) -> int:
        return 4 * n if self.max_iter is None else self.max_iter


@dataclass(frozen=True)
class SolveResult:
    x: Vector
    method: str
    sketch: str | None
    d: int | None
    iterations: int
    residual_norm: float
    termination: str
    wall_time_s: float


def _operator_spec(spec: SketchSpec | None, method: str, m: int, n: int,
                   d_factor: float) -> SketchSpec:
    """d from d_factor, seed mixed with the method tag (solvers.py:273-279)."""
    if spec is None:
        spec = SketchSpec(kind=DEFAULT_KIND, embed_dim=1)
    d = default_embed_dim(m, n, d_factor)
    return replace(spec, embed_dim=d, seed=derive_seed(spec.seed, method))


def _residual_device(A: Matrix, A_dev, lda: int, b_dev, x_dev) -> float:
    out = np.zeros(1, dtype=np.float64)
    if isinstance(A, SparseMatrix):
        indptr, indices, values = A.device_arrays()
        _native.call("skl_residual_csr", _native.ptr(indptr), _native.ptr(indices),
                     _native.ptr(values), A.rows, A.cols, _native.ptr(x_dev), _native.ptr(b_dev),
                     _native.ptr(out), current_stream())
    else:
        _native.call("skl_residual_dense", _native.ptr(A_dev), A.rows, A.cols, lda,
                     _native.ptr(x_dev), _native.ptr(b_dev), _native.ptr(out), current_stream())
    return float(out[0])


def sketch_operands_device(op, A: Matrix, b: Vector):
    """(SA, Sb, A_dev, lda, b_dev) on the device for one SAA solve; A and b
    are uploaded once when host-resident and reused for the residual."""
    if isinstance(A, SparseMatrix):
        b_dev = b.data if b.on_device else to_device(b.data)
        if op.kind in ("countsketch", "sparsesign"):
            SA = _countsketch_csr_device(op, A)
            Sb = _apply_dense_tensor(op, b_dev.reshape(-1, 1), A.rows, 1, lda=A.rows).reshape(-1)
            return SA, Sb, None, 0, b_dev
        dense = to_device(np.asfortranarray(A.to_scipy().toarray()))
        SA = _apply_dense_tensor(op, dense, A.rows, A.cols, lda=A.rows)
        Sb = _apply_dense_tensor(op, b_dev.reshape(-1, 1), A.rows, 1, lda=A.rows).reshape(-1)
        return SA, Sb, None, 0, b_dev
    if (not A.on_device and not b.on_device and op.kind == "countsketch"
            and not _few_long_columns(A.rows, A.cols + 1)):
        # host A: row blocks stream to the device under the sketch kernel and
        # land in a device copy kept for the residual pass (one H2D of A)
        m, n, d = A.rows, A.cols, op.target_dim
        ld = (m + 1) // 2 * 2
        A_dev = device_f64((m, n), fortran=True, ld=ld)
        b_dev = device_f64((m,))
        SA = device_f64((d, n), fortran=True)
        Sb = device_f64((d,))
        op.device_plan().apply_host(A.data, m, n, m, np.ascontiguousarray(b.data), SA, d, Sb,
                                    A_keep=A_dev, ld_keep=ld, b_keep=b_dev)
        return SA, Sb, A_dev, ld, b_dev
    b_dev = b.data if b.on_device else to_device(b.data)
    A_dev = A.data if A.on_device else to_device(A.data)
    lda = A.ld if A.on_device else A.rows
    if op.kind in ("countsketch", "sparsesign"):
        SA, Sb = _countsketch_dense_device(op, A_dev, lda, A.cols, b=b_dev)
    elif op.kind == "srht":
        SA, Sb = _srht_device_ab(op, A_dev, lda, A.cols, b_dev.contiguous())
    else:
        SA = _apply_dense_tensor(op, A_dev, A.rows, A.cols, lda=lda)
        Sb = _apply_dense_tensor(op, b_dev.reshape(-1, 1), A.rows, 1, lda=A.rows).reshape(-1)
    return SA, Sb, A_dev, lda, b_dev


_EVENTS = threading.local()


def _timing_events():
    """A per-thread, per-device pair of timing events for wall_time_s (creating
    two events on every solve cost host time ahead of the first launch)."""
    dev = torch.cuda.current_device()
    pairs = getattr(_EVENTS, "pairs", None)
    if pairs is None:
        pairs = _EVENTS.pairs = {}
    ev = pairs.get(dev)
    if ev is None:
        ev = pairs[dev] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    return ev


def sketch_and_apply(problem: LeastSquaresProblem, spec: SketchSpec | None = None,
                     opts: SolverOptions | None = None) -> SolveResult:
    """Solve min ||S A x - S b|| by QR, one shot (solvers.py:296-320)."""
    A, b = problem.A, problem.b
    if A.rows < A.cols:
        raise ShapeError(f"need rows >= cols, got {A.rows}x{A.cols}")
    require_cuda()
    opts = opts or SolverOptions()
    op_spec = _operator_spec(spec, "saa", A.rows, A.cols, opts.d_factor)
    t0 = time.perf_counter()
    if opts.devices is not None and len(opts.devices) > 1:
        return _sketch_and_apply_devices(A, b, op_spec, opts.devices, t0)
    if opts.devices is not None:
        with torch.cuda.device(opts.devices[0]):
            return sketch_and_apply(problem, spec, replace(opts, devices=None))
    # The factorisation is enqueued without its own synchronisation and its
    # rank flag checked after the residual pass (one host round trip per
    # solve); wall_time_s still covers sketch + QR + back-solve, as the
    # reference's, through events on the stream.
    ev0, ev1 = _timing_events()
    ev0.record()
    op = build_sketch(op_spec, A.rows)
    SA, Sb, A_dev, lda, b_dev = sketch_operands_device(op, A, b)
    d = op.target_dim
    x_dev, rank_check = qr_solve_device_async(SA, d, Sb, d, A.cols)
    ev1.record()
    rnorm = _residual_device(A, A_dev, lda, b_dev, x_dev)
    try:
        x_fix = rank_check()
    except SingularFactorError as exc:
        raise SingularFactorError(
            f"sketched matrix ({op_spec.kind}, d={d}) is rank deficient: {exc}; "
            f"a larger embedding dimension may help") from exc
    if x_fix is not None:  # the CholeskyQR path handed over to Householder
        x_dev = x_fix
        rnorm = _residual_device(A, A_dev, lda, b_dev, x_dev)
    wall = ev0.elapsed_time(ev1) * 1e-3
    x = x_dev if (isinstance(A, DenseMatrix) and A.on_device) else x_dev.cpu().numpy()
    return SolveResult(x=Vector._of_solution(x, rnorm), method="saa", sketch=op_spec.kind, d=d,
                       iterations=0, residual_norm=rnorm, termination="direct", wall_time_s=wall)


def _sketch_and_apply_devices(A: Matrix, b: Vector, op_spec: SketchSpec, devices, t0: float):
    """SAA with A's rows sharded over several devices (multidevice.py); the
    operator is the global one (same hashes/signs/samples as one device)."""
    from .multidevice import sketch_and_apply_devices

    with torch.cuda.device(devices[0]):
        op = build_sketch(op_spec, A.rows)
        d = op.target_dim
        try:
            x_dev, rnorm = sketch_and_apply_devices(op, A, b, devices)
        except SingularFactorError as exc:
            raise SingularFactorError(
                f"sketched matrix ({op_spec.kind}, d={d}) is rank deficient: {exc}; "
                f"a larger embedding dimension may help") from exc
        wall = time.perf_counter() - t0
        x = x_dev if (isinstance(A, DenseMatrix) and A.on_device) else x_dev.cpu().numpy()
    return SolveResult(x=Vector._of_solution(x, rnorm), method="saa", sketch=op_spec.kind, d=d,
                       iterations=0, residual_norm=rnorm, termination="direct", wall_time_s=wall)


def _operator_device(A: Matrix):
    """(LSQR operator, dense device A or None, lda) for a carrier."""
    from ._lsqr import CsrOperator, DenseOperator

    if isinstance(A, SparseMatrix):
        return CsrOperator(A), None, 0
    A_dev = A.data if A.on_device else to_device(A.data)
    lda = A.ld if A.on_device else A.rows
    if A_dev.data_ptr() % 16 or (lda % 2 and A.cols > 1):
        from .sketch import _aligned

        A_dev, lda = _aligned(A_dev, lda, A.cols)
    return DenseOperator(A_dev, lda, A.rows, A.cols), A_dev, lda


def _lsqr_result(A, b_dev, A_dev, lda, x_dev, itn, istop, method, sketch, d, t0):
    wall = time.perf_counter() - t0
    rnorm = _residual_device(A, A_dev, lda, b_dev, x_dev)
    x = x_dev if (isinstance(A, DenseMatrix) and A.on_device) else x_dev.cpu().numpy()
    return SolveResult(x=Vector._of_solution(x, rnorm), method=method, sketch=sketch, d=d,
                       iterations=itn, residual_norm=rnorm, termination="max_iter" if istop == 7 else "atol_btol",
                       wall_time_s=wall)


def _precond_device(R: DenseMatrix, n: int):
    """Validate a user preconditioner as the reference does (solvers.py:137-145)
    and return it column-major on the device."""
    if R.rows != R.cols or R.cols != n:
        raise ShapeError(f"preconditioner must be {n}x{n}, got {R.rows}x{R.cols}")
    r = R.to_numpy()
    if np.any(np.tril(r, -1) != 0.0):
        raise ShapeError("preconditioner must be upper triangular")
    zero = np.flatnonzero(np.diagonal(r) == 0.0)
    if zero.size:
        raise SingularFactorError(f"zero diagonal entry at index {int(zero[0])}")
    require_cuda()
    return to_device(np.asfortranarray(r))


def lsqr(A: Matrix, b: Vector, opts: SolverOptions | None = None,
         precond_R: DenseMatrix | None = None, callback=None) -> SolveResult:
    """LSQR on the device (solvers.py:110-255): plain, or right-preconditioned
    by an upper-triangular ``precond_R`` (the iteration runs on A R^-1 and the
    result is x = R^-1 y); ``callback(itn, iterate, rnorm)`` once per
    iteration, as in the reference."""
    from ._lsqr import lsqr_device

    if b.len != A.rows:
        raise ShapeError(f"A is {A.rows}x{A.cols} but b has length {b.len}")
    opts = opts or SolverOptions()
    R_dev = _precond_device(precond_R, A.cols) if precond_R is not None else None
    require_cuda()
    t0 = time.perf_counter()
    lop, A_dev, lda = _operator_device(A)
    b_dev = b.data if b.on_device else to_device(b.data)
    x, itn, istop = lsqr_device(lop, A.rows, A.cols, b_dev, opts.atol, opts.btol,
                                opts.resolve_max_iter(A.cols), R=R_dev,
                                ldr=A.cols if R_dev is not None else 0, callback=callback)
    return _lsqr_result(A, b_dev, A_dev, lda, x, itn, istop, "lsqr", None, None, t0)


def sketch_and_precondition(problem: LeastSquaresProblem, spec: SketchSpec | None = None,
                            opts: SolverOptions | None = None) -> SolveResult:
    """LSQR right-preconditioned by R from QR(S A), warm-started from the
    sketched solution (solvers.py:323-361)."""
    from ._lsqr import lsqr_device

    A, b = problem.A, problem.b
    if A.rows < A.cols:
        raise ShapeError(f"need rows >= cols, got {A.rows}x{A.cols}")
    require_cuda()
    opts = opts or SolverOptions()
    op_spec = _operator_spec(spec, "sap", A.rows, A.cols, opts.d_factor)
    t0 = time.perf_counter()
    lop, A_dev, lda = _operator_device(A)
    op = build_sketch(op_spec, A.rows)
    A_sk = A if (isinstance(A, SparseMatrix) or A.on_device) else DenseMatrix(A_dev)
    SA, Sb, _, _, b_dev = sketch_operands_device(op, A_sk, b)
    d, n = op.target_dim, A.cols
    try:
        x0, R, _ = qr_solve_device(SA, d, Sb, d, n, want_r=True)
    except SingularFactorError as exc:
        raise SingularFactorError(
            f"sketched matrix ({op_spec.kind}, d={d}) is rank deficient: {exc}; "
            f"a larger embedding dimension may help") from exc
    max_iter = opts.resolve_max_iter(n)
    if opts.warm_start:
        # r0 = b - A x0 (solvers.py:345-349): -(A x0) - (-1) b
        r0 = device_f64((A.rows,))
        scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
        from ._lsqr import _Workspace

        lop.mv(x0, -1.0, -1.0, b_dev, r0, scratch, _Workspace(A.rows, n), current_stream())
        xi, itn, istop = lsqr_device(lop, A.rows, n, r0, opts.atol, opts.btol, max_iter,
                                     R=R, ldr=n)
        x = x0 + xi
    else:
        x, itn, istop = lsqr_device(lop, A.rows, n, b_dev, opts.atol, opts.btol, max_iter,
                                    R=R, ldr=n)
    return _lsqr_result(A, b_dev, A_dev, lda, x, itn, istop, "sap", op_spec.kind, d, t0)


def direct(problem: LeastSquaresProblem) -> SolveResult:
    """The ``direct`` method: Householder QR of A itself on the device and
    x = R^-1 Q^T b (solvers.py:381-396 via linalg.py:221-232
    ``normal_equations_oracle``); sparse A is densified on the device first."""
    A, b = problem.A, problem.b
    if b.len != A.rows:
        raise ShapeError(f"A is {A.rows}x{A.cols} but b has length {b.len}")
    if A.rows < A.cols:
        raise ShapeError(f"need rows >= cols, got {A.rows}x{A.cols}")
    require_cuda()
    t0 = time.perf_counter()
    b_dev = b.data if b.on_device else to_device(b.data)
    if isinstance(A, SparseMatrix):
        indptr, indices, values = A.device_arrays()
        rows = torch.repeat_interleave(
            torch.arange(A.rows, device="cuda"), indptr[1:] - indptr[:-1])
        dense = torch.zeros((A.cols, A.rows), dtype=torch.float64, device="cuda")
        dense[indices, rows] = values  # column-major m x n: row j of dense is column j
        A_dev, lda = dense.t(), A.rows
    else:
        A_dev = A.data if A.on_device else to_device(A.data)
        lda = A.ld if A.on_device else A.rows
    x_dev, _, _ = qr_solve_device(A_dev, lda, b_dev, A.rows, A.cols)
    wall = time.perf_counter() - t0
    if isinstance(A, SparseMatrix):
        rnorm = _residual_device(A, None, 0, b_dev, x_dev)
    else:
        rnorm = _residual_device(A, A_dev, lda, b_dev, x_dev)
    x = x_dev if (isinstance(A, DenseMatrix) and A.on_device) else x_dev.cpu().numpy()
    return SolveResult(x=Vector(x), method="direct", sketch=None, d=None, iterations=0,
                       residual_norm=rnorm, termination="direct", wall_time_s=wall)


_SIDE = threading.local()


def _side_streams():
    """Two non-blocking streams per device (per thread) for solve_many."""
    dev = torch.cuda.current_device()
    per = getattr(_SIDE, "streams", None)
    if per is None:
        per = _SIDE.streams = {}
    st = per.get(dev)
    if st is None:
        st = per[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return st


def solve_many(problems, method: str = "saa", spec: SketchSpec | None = None,
               opts: SolverOptions | None = None) -> list[SolveResult]:
    """Independent solves, each the same as solve(problem, method, spec,
    opts) (bitwise: the same kernels on the same data), enqueued back to
    back on two streams with one host synchronisation for the batch.  On the
    B200 the reduced solve of problem i (a latency-bound chain on a few SMs)
    then runs beside the HBM-bound sketch and residual passes of its
    neighbours instead of leaving the other SMs idle, and the host-side
    turnaround between solves disappears.  Sketch-and-apply on one device is
    batched; other methods and device lists run one solve at a time."""
    problems = list(problems)
    opts = opts or SolverOptions()
    if method != "saa" or (opts.devices is not None and len(opts.devices) > 1):
        return [solve(p, method, spec, opts) for p in problems]
    if opts.devices is not None:
        with torch.cuda.device(opts.devices[0]):
            return solve_many(problems, method, spec, replace(opts, devices=None))
    require_cuda()
    if not problems:
        return []
    caller = torch.cuda.current_stream()
    streams = _side_streams()
    pinned = torch.zeros((len(problems), 3), dtype=torch.float64, pin_memory=True)
    work = []
    for i, prob in enumerate(problems):
        A, b = prob.A, prob.b
        if A.rows < A.cols:
            raise ShapeError(f"need rows >= cols, got {A.rows}x{A.cols}")
        op_spec = _operator_spec(spec, "saa", A.rows, A.cols, opts.d_factor)
        st = streams[i & 1]
        st.wait_stream(caller)
        with torch.cuda.stream(st):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            op = build_sketch(op_spec, A.rows)
            SA, Sb, A_dev, lda, b_dev = sketch_operands_device(op, A, b)
            d = op.target_dim
            x_dev, check = qr_solve_device_async(SA, d, Sb, d, A.cols, flags=pinned[i, :2])
            ev1.record()
            out = pinned[i, 2:]
            if isinstance(A, SparseMatrix):
                indptr, indices, values = A.device_arrays()
                _native.call("skl_residual_csr_async", _native.ptr(indptr), _native.ptr(indices),
                             _native.ptr(values), A.rows, A.cols, _native.ptr(x_dev),
                             _native.ptr(b_dev), out.data_ptr(), current_stream())
            else:
                _native.call("skl_residual_dense_async", _native.ptr(A_dev), A.rows, A.cols, lda,
                             _native.ptr(x_dev), _native.ptr(b_dev), out.data_ptr(),
                             current_stream())
            work.append((prob, op_spec, d, SA, Sb, A_dev, lda, b_dev, x_dev, check, ev0, ev1, st))
    for st in streams:
        caller.wait_stream(st)
    for st in streams:
        st.synchronize()
    results = []
    for i, (prob, op_spec, d, SA, Sb, A_dev, lda, b_dev, x_dev, check, ev0, ev1, st) in enumerate(work):
        A = prob.A
        with torch.cuda.stream(st):
            try:
                x_fix = check()
            except SingularFactorError as exc:
                raise SingularFactorError(
                    f"sketched matrix ({op_spec.kind}, d={d}) is rank deficient: {exc}; "
                    f"a larger embedding dimension may help") from exc
            rnorm = float(pinned[i, 2])
            if x_fix is not None:  # the CholeskyQR path handed over to Householder
                x_dev = x_fix
                rnorm = _residual_device(A, A_dev, lda, b_dev, x_dev)
        wall = ev0.elapsed_time(ev1) * 1e-3
        if isinstance(A, DenseMatrix) and A.on_device:
            x_dev.record_stream(caller)  # handed to the caller's stream
            x = x_dev
        else:
            x = x_dev.cpu().numpy()
        results.append(SolveResult(x=Vector._of_solution(x, rnorm), method="saa",
                                   sketch=op_spec.kind, d=d, iterations=0, residual_norm=rnorm,
                                   termination="direct", wall_time_s=wall))
    return results


def solve(problem: LeastSquaresProblem, method: str = "lsqr", spec: SketchSpec | None = None,
          opts: SolverOptions | None = None) -> SolveResult:
    """Dispatch (solvers.py:364-398); wall_time_s covers the full path.

    Same default as the reference (``method="lsqr"``).  Every method runs on
    the device, for dense and CSR operands."""
    if method not in METHODS:
        raise SpecError(f"unknown method {method!r}, expected one of {METHODS}")
    t0 = time.perf_counter()
    if method == "saa":
        result = sketch_and_apply(problem, spec, opts)
    elif method == "sap":
        result = sketch_and_precondition(problem, spec, opts)
    elif method == "lsqr":
        result = lsqr(problem.A, problem.b, opts)
    else:
        result = direct(problem)
    wall = time.perf_counter() - t0
    return replace(result, wall_time_s=wall)
