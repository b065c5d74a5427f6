"""Device LSQR (Paige & Saunders), plain or right-preconditioned by R.

Mirrors /root/reference/pkg/src/sketchls/solvers.py:110-255 (`lsqr`) and
:258-270 (`_sym_ortho`).  The vector work runs in the fused kernels of
csrc/skl_lsqr.cu (one HBM pass over dense A per iteration for n <= 256,
two otherwise; the n x n triangular solves with R in one CTA each); the scalar recurrence -- Givens
rotations, the ||A|| estimate and the five stopping rules -- is the
reference's code, line for line, on host floats read back once per step.
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import _native
from ._device import current_stream, device_f64, require_cuda, torch
from .errors import NumericalBreakdownError

_EPS = float(np.finfo(np.float64).eps)  # solvers.py:37


def sym_ortho(a: float, b: float) -> tuple[float, float, float]:
    """Stable Givens rotation (c, s, r) with c*a + s*b = r (solvers.py:258-270)."""
    if b == 0.0:
        return math.copysign(1.0, a) if a != 0 else 1.0, 0.0, abs(a)
    if a == 0.0:
        return 0.0, math.copysign(1.0, b), abs(b)
    if abs(b) > abs(a):
        tau = a / b
        s = math.copysign(1.0, b) / math.sqrt(1.0 + tau * tau)
        return s * tau, s, b / s
    tau = b / a
    c = math.copysign(1.0, a) / math.sqrt(1.0 + tau * tau)
    return c, c * tau, a / c


class DenseOperator:
    """x -> A x and u -> A^T u for column-major device A (m x n, ld lda)."""

    def __init__(self, A, lda: int, m: int, n: int):
        self.A, self.lda, self.m, self.n = A, lda, m, n

    def mv(self, y, s, alpha, u_in, u_out, norm2, ws, st):
        _native.call("skl_lsqr_gemv_n", _native.ptr(self.A), self.m, self.n, self.lda,
                     _native.ptr(y), s, alpha, _native.ptr(u_in), _native.ptr(u_out),
                     _native.ptr(norm2), _native.ptr(ws.work), _native.ptr(ws.counters), st)

    def rmv(self, u_raw, beta, u_n, z, ws, st):
        _native.call("skl_lsqr_gemv_t", _native.ptr(self.A), self.m, self.n, self.lda,
                     _native.ptr(u_raw), beta, _native.ptr(u_n), _native.ptr(z),
                     _native.ptr(ws.work), _native.ptr(ws.counters), st)

    def fusable(self) -> bool:
        """Both products in one pass (skl_lsqr_fused): n <= 256, A 16-byte
        aligned with an even leading dimension."""
        return (self.n <= 256 and self.lda % 2 == 0 and self.A.data_ptr() % 16 == 0
                and not os.environ.get("SKL_LSQR_TWO_PASS"))

    def fused(self, y, alpha, r_prev, beta_prev, r_out, z, norm2, work, ws, st):
        _native.call("skl_lsqr_fused", _native.ptr(self.A), self.m, self.n, self.lda,
                     _native.ptr(y), 1.0, alpha, _native.ptr(r_prev), beta_prev,
                     _native.ptr(r_out), _native.ptr(z), _native.ptr(norm2), _native.ptr(work),
                     _native.ptr(ws.counters), st)


class CsrOperator:
    """The same two products for a CSR matrix (SparseMatrix device arrays).
    A^T u runs on the CSC form, built once on the device: a stable sort of
    the nonzeros by column keeps each column's rows ascending, so the
    transposed product is deterministic."""

    def __init__(self, A):
        self.indptr, self.indices, self.values = A.device_arrays()
        self.m, self.n = A.rows, A.cols
        self.colptr, self.rowidx, self.cval = A.device_csc()  # cached with the operand

    def mv(self, y, s, alpha, u_in, u_out, norm2, ws, st):
        _native.call("skl_lsqr_spmv", _native.ptr(self.indptr), _native.ptr(self.indices),
                     _native.ptr(self.values), self.m, _native.ptr(y), s, alpha,
                     _native.ptr(u_in), _native.ptr(u_out), _native.ptr(norm2),
                     _native.ptr(ws.work), _native.ptr(ws.counters), st)

    def rmv(self, u_raw, beta, u_n, z, ws, st):
        _native.call("skl_lsqr_csc_t", _native.ptr(self.colptr), _native.ptr(self.rowidx),
                     _native.ptr(self.cval), self.m, self.n, _native.ptr(u_raw), beta,
                     _native.ptr(u_n), _native.ptr(z), st)


class _Workspace:
    def __init__(self, m: int, n: int):
        self.u_raw = device_f64((m,))
        self.u = device_f64((m,))
        self.z = device_f64((n,))
        self.v = device_f64((n,))
        self.v_raw = device_f64((n,))
        self.y = device_f64((n,))
        self.w = device_f64((n,))
        self.x = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.scal = torch.zeros(4, dtype=torch.float64, device="cuda")  # beta2, alfa2, x2
        nw = int(_native.lib().skl_lsqr_work_size(m, n))
        nc = int(_native.lib().skl_lsqr_counter_size(n))
        self.work = device_f64((nw,))
        self.counters = torch.zeros(nc, dtype=torch.int32, device="cuda")


# indices of the device-side recurrence state (csrc/skl_lsqr.cu, LS_*)
_LS_BETA2, _LS_ALFA2, _LS_XNORM2, _LS_ALFA, _LS_BETA = 0, 1, 2, 3, 4
_LS_RHOBAR, _LS_PHIBAR, _LS_ANORM, _LS_RNORM, _LS_ARNORM, _LS_BPREV = 5, 6, 7, 10, 11, 12


def _lsqr_device_driven(op, ws, fwork, n, Rp, ldr, Rinv, alfa, beta, atol, btol, max_iter, R,
                        trsv_n, callback, st):
    """The fused-pass LSQR loop with the scalar recurrence on the device
    (skl_lsqr_step_dev): per iteration one D2H read of the state, taken
    while the next iteration's pass over A already runs (it does not depend
    on the stopping decision, and if the loop stops its result is unused).
    The recurrence performs the host loop's IEEE operations in the same
    order, so iterates, iteration counts and stopping rule are the same."""
    P = _native.ptr
    # R^{-1} in full once (n <= 256): the step's two triangular solves become
    # products with it (SKL_LSQR_BLOCK_SOLVES=1 keeps the blocked solves)
    RF = None
    if Rp is not None and Rinv is not None and n <= 256 and not os.environ.get(
            "SKL_LSQR_BLOCK_SOLVES"):
        RF = device_f64((n * n,))
        _native.call("skl_lsqr_rinv_full", Rp, ldr, n, P(RF), st)
    nst = int(_native.lib().skl_lsqr_state_size())
    state = torch.zeros(nst, dtype=torch.float64, device="cuda")
    init = torch.zeros(nst, dtype=torch.float64)
    init[_LS_ALFA], init[_LS_RHOBAR], init[_LS_PHIBAR], init[_LS_BPREV] = alfa, alfa, beta, beta
    state.copy_(init)
    rep = torch.empty(nst, dtype=torch.float64, pin_memory=True)
    done = torch.cuda.Event()
    bnorm = beta
    r_prev, r_out = ws.u_raw, ws.u

    def enqueue_pass(rp, ro):
        _native.call("skl_lsqr_fused_dev", P(op.A), op.m, op.n, op.lda, P(ws.y), P(rp), P(ro),
                     P(ws.z), state.data_ptr() + 8 * _LS_BETA2, P(fwork), P(ws.counters),
                     P(state), st)

    enqueue_pass(r_prev, r_out)
    itn = istop = 0
    while itn < max_iter:
        itn += 1
        if RF is not None:
            _native.call("skl_lsqr_step_full_dev", P(RF), n, P(ws.z), P(ws.v), P(ws.v_raw),
                         P(ws.y), P(ws.w), P(ws.x), P(state), st)
        else:
            _native.call("skl_lsqr_step_dev", Rp, ldr, n, P(Rinv), P(ws.z), P(ws.v), P(ws.v_raw),
                         P(ws.y), P(ws.w), P(ws.x), P(state), st)
        rep.copy_(state, non_blocking=True)
        done.record()
        r_prev, r_out = r_out, r_prev
        if itn < max_iter:
            enqueue_pass(r_prev, r_out)  # the next pass overlaps the host's read
        done.synchronize()
        s_ = rep.tolist()
        alfa, beta = s_[_LS_ALFA], s_[_LS_BETA]
        anorm, rnorm, arnorm = s_[_LS_ANORM], s_[_LS_RNORM], s_[_LS_ARNORM]
        if not (math.isfinite(alfa) and math.isfinite(beta)):
            raise NumericalBreakdownError(
                f"non-finite bidiagonalization coefficient at iteration {itn}")
        xnorm = math.sqrt(s_[_LS_XNORM2])
        if not math.isfinite(rnorm):
            raise NumericalBreakdownError(f"non-finite residual estimate at iteration {itn}")
        if callback is not None:
            callback(itn, ws.x.cpu().numpy(), rnorm)
        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm + _EPS)
        t1 = test1 / (1.0 + anorm * xnorm / bnorm)
        rtol = btol + atol * anorm * xnorm / bnorm
        if itn >= max_iter:
            istop = 7
        if 1.0 + test2 <= 1.0:
            istop = 5
        if 1.0 + t1 <= 1.0:
            istop = 4
        if test2 <= atol:
            istop = 2
        if test1 <= rtol:
            istop = 1
        if istop != 0:
            break
    x = ws.x
    if R is not None:
        xr = device_f64((n,))
        tmp = ws.x.clone()
        trsv_n(0.0, tmp, xr)
        x = xr
    return x, itn, istop


def lsqr_device(op, m: int, n: int, b, atol: float, btol: float, max_iter: int,
                R=None, ldr: int = 0, callback=None):
    """LSQR on the device for the operator ``op`` (DenseOperator or
    CsrOperator, m x n) and b (device tensor).  With R (n x n upper,
    column-major) the iteration runs on y -> A R^-1 y and returns x = R^-1 y
    (solvers.py:146-151, 241).  ``callback(itn, iterate, rnorm)`` is called
    once per iteration with a host copy of the iterate (y when
    preconditioned) and the recurrence residual estimate (solvers.py:220-221).
    Returns (x tensor, iterations, istop)."""
    require_cuda()
    ws = _Workspace(m, n)
    st = current_stream()
    P = _native.ptr
    Rp = P(R) if R is not None else None
    sc = ws.scal
    # R is fixed for the whole solve: invert its 32 x 32 diagonal blocks once
    # and let every triangular solve use them (SKL_LSQR_DTRTRS=1 keeps the
    # per-element dtrsv substitution order instead)
    Rinv = None
    if R is not None and not os.environ.get("SKL_LSQR_DTRTRS"):
        Rinv = device_f64((((n + 31) // 32) * 1024,))
        _native.call("skl_lsqr_rinv_blocks", Rp, ldr, n, P(Rinv), st)

    def trsv_t(z, beta_, v_prev, v_out, norm2):
        if Rinv is not None:
            _native.call("skl_lsqr_trsv_t_inv", Rp, ldr, n, P(Rinv), P(z), beta_, P(v_prev),
                         P(v_out), P(norm2), st)
        else:
            _native.call("skl_lsqr_trsv_t", Rp, ldr, n, P(z), beta_, P(v_prev), P(v_out),
                         P(norm2), st)

    def trsv_n(alfa_, v, y):
        if Rinv is not None:
            _native.call("skl_lsqr_trsv_n_inv", Rp, ldr, n, P(Rinv), alfa_, P(v), P(y), st)
        else:
            _native.call("skl_lsqr_trsv_n", Rp, ldr, n, alfa_, P(v), P(y), st)

    def read(i: int) -> float:
        return float(sc[i].item())

    # u = b; beta = ||u||  (u_out = -(-1) b: an exact copy plus its norm)
    _native.call("skl_lsqr_gemv_n", None, m, 0, m, None, 0.0, -1.0, P(b), P(ws.u_raw),
                 P(sc[0:1]), P(ws.work), P(ws.counters), st)
    beta = math.sqrt(read(0))
    alfa = 0.0
    if beta > 0:
        # u /= beta; v = rmv(u); alfa = ||v||
        op.rmv(ws.u_raw, beta, ws.u, ws.z, ws, st)
        ws.v.zero_()
        trsv_t(ws.z, 0.0, ws.v, ws.v_raw, sc[1:2])
        alfa = math.sqrt(read(1))
    else:
        ws.u.copy_(ws.u_raw)
        ws.v_raw.zero_()
    # v /= alfa (if alfa > 0); y = R^-1 v; w = v
    trsv_n(alfa, ws.v_raw, ws.y)
    ws.v.copy_(ws.v_raw)
    ws.w.copy_(ws.v)

    itn = istop = 0
    anorm = 0.0
    rhobar, phibar, bnorm = alfa, beta, beta
    if alfa * beta == 0.0:
        return ws.x, 0, 0  # b or A^T b is zero: x = 0 exactly (solvers.py:176-189)

    # one pass over A per step where the operator allows it: u = r_prev /
    # beta_prev is formed inside the pass, A^T u comes out of the same pass
    fused = isinstance(op, DenseOperator) and op.fusable()
    if fused:
        fwork = device_f64((int(_native.lib().skl_lsqr_fused_work_size(n)),))
        r_prev, r_out, beta_prev = ws.u_raw, ws.u, beta
        if not os.environ.get("SKL_LSQR_HOST_LOOP"):
            return _lsqr_device_driven(op, ws, fwork, n, Rp, ldr, Rinv, alfa, beta, atol, btol,
                                       max_iter, R, trsv_n, callback, st)

    while itn < max_iter:
        itn += 1
        if fused:
            # u = r_prev / beta_prev ; r = mv(v) - alfa u ; beta = ||r|| ; z = rmv(r / beta)
            op.fused(ws.y, alfa, r_prev, beta_prev, r_out, ws.z, sc[0:1], fwork, ws, st)
            beta = math.sqrt(read(0))
            r_prev, r_out = r_out, r_prev
            beta_prev = beta if beta > 0 else 1.0  # u stays unnormalised (solvers.py:193)
        else:
            # u = mv(v) - alfa u ; beta = ||u||
            op.mv(ws.y, 1.0, alfa, ws.u, ws.u_raw, sc[0:1], ws, st)
            beta = math.sqrt(read(0))
        if beta > 0:
            anorm = math.sqrt(anorm**2 + alfa**2 + beta**2)
            # u /= beta ; v = rmv(u) - beta v ; alfa = ||v|| ; v /= alfa
            if not fused:
                op.rmv(ws.u_raw, beta, ws.u, ws.z, ws, st)
            trsv_t(ws.z, beta, ws.v, ws.v_raw, sc[1:2])
            alfa = math.sqrt(read(1))
            trsv_n(alfa, ws.v_raw, ws.y)
            ws.v, ws.v_raw = ws.v_raw, ws.v
        elif not fused:
            ws.u, ws.u_raw = ws.u_raw, ws.u  # u stays unnormalised (solvers.py:193)
        if not (math.isfinite(alfa) and math.isfinite(beta)):
            raise NumericalBreakdownError(
                f"non-finite bidiagonalization coefficient at iteration {itn}")

        cs, sn, rho = sym_ortho(rhobar, beta)
        theta = sn * alfa
        rhobar = -cs * alfa
        phi = cs * phibar
        phibar = sn * phibar

        # x += (phi/rho) w ; w = v + (-theta/rho) w ; xnorm = ||x||
        _native.call("skl_lsqr_xw", n, phi / rho, -theta / rho, P(ws.v), P(ws.w), P(ws.x),
                     P(sc[2:3]), st)
        rnorm = phibar
        arnorm = alfa * abs(sn * phi)
        xnorm = math.sqrt(read(2))
        if not math.isfinite(rnorm):
            raise NumericalBreakdownError(f"non-finite residual estimate at iteration {itn}")
        if callback is not None:
            callback(itn, ws.x.cpu().numpy(), rnorm)

        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm + _EPS)
        t1 = test1 / (1.0 + anorm * xnorm / bnorm)
        rtol = btol + atol * anorm * xnorm / bnorm
        if itn >= max_iter:
            istop = 7
        if 1.0 + test2 <= 1.0:
            istop = 5
        if 1.0 + t1 <= 1.0:
            istop = 4
        if test2 <= atol:
            istop = 2
        if test1 <= rtol:
            istop = 1
        if istop != 0:
            break

    x = ws.x
    if R is not None:
        xr = device_f64((n,))
        tmp = ws.x.clone()
        trsv_n(0.0, tmp, xr)
        x = xr
    return x, itn, istop
