"""CPU ORACLE -- test infrastructure only.

A numpy/scipy restatement of the reference's hot path
(/root/reference/pkg/src/sketchls, package `sketchls`), used as the
checker by tests/, by `__graft_entry__.smoke()` and as the `cpu_baseline`
/ `--impl reference` arm of bench.py.  Nothing in the product package
imports this module; the product path fails loudly without its CUDA
library instead of falling back here.

Pinning: every function is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports /root/reference in
the build container; tests/test_oracle_golden.py compares).  The random
draws live in a third-party dependency, numpy 2.3.5 (Philox4x64-10,
Lemire bounded integers, Fisher-Yates permutation, 256-level ziggurat);
`oracle/c/philox_oracle.c` restates that published algorithm in plain C
and is pinned against numpy's own output.  The CountSketch arithmetic
lives in scipy 1.18.1 sparsetools (`csr_matvecs`: per bucket, ascending
source rows, folded from +0.0), the Gaussian in BLAS dgemm, the QR in
LAPACK dgeqrf/dorgqr; the restatement calls the same routines the
reference calls, in the same order.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg
import scipy.sparse

MASK64 = (1 << 64) - 1
RANK_TOL = 1e-14  # linalg.py:23


def splitmix64(z: int) -> int:
    """rng.py:19-24."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_seed(seed: int, *tags) -> int:
    """rng.py:27-40."""
    state = splitmix64(seed & MASK64)
    for tag in tags:
        if isinstance(tag, str):
            for byte in tag.encode("utf-8"):
                state = splitmix64(state ^ byte)
        else:
            state = splitmix64(state ^ (int(tag) & MASK64))
    return state


def stream(key: int) -> np.random.Generator:
    """rng.py:43-45 (numpy 2.3.5 Philox)."""
    return np.random.Generator(np.random.Philox(key=key & MASK64))


def default_embed_dim(m: int, n: int, d_factor: float = 4.0) -> int:
    """sketch.py:41-45."""
    return min(m, max(n, math.ceil(d_factor * n)))


def operator_key(seed: int, kind: str, m: int, method: str | None = None) -> int:
    """Key of the operator stream: sketch.py:93, preceded by the method tag
    of solvers.py:279 when built by a solver."""
    if method is not None:
        seed = derive_seed(seed, method)
    return derive_seed(seed, kind, m)


# ------------------------------------------------------------------ draws
def countsketch_draws(key: int, m: int, d: int):
    """sketch.py:97-99 -> (rows int64, signs float64)."""
    rng = stream(key)
    rows = rng.integers(0, d, size=m)
    signs = 2.0 * rng.integers(0, 2, size=m) - 1.0
    return rows, signs


def srht_draws(key: int, m: int, d: int):
    """sketch.py:116-127 -> (sign_diag float64 [m_pad], row_sample int64 [d], m_pad)."""
    rng = stream(key)
    m_pad = 1 << (m - 1).bit_length()
    signs = (2.0 * rng.integers(0, 2, size=m_pad) - 1.0).astype(np.float64)
    row_sample = np.ascontiguousarray(rng.permutation(m_pad)[:d], dtype=np.int64)
    return signs, row_sample, m_pad


def gaussian_draws(key: int, d: int, m: int) -> np.ndarray:
    """sketch.py:94-96 -> C-order d x m."""
    return stream(key).standard_normal((d, m)) / math.sqrt(d)


# ------------------------------------------------------------------ applies
def sparsesign_draws(key: int, m: int, d: int, s: int):
    """sketch.py:104-110, 130-149: (rows (m, s) int64, signs (m, s) +-1.0)."""
    rng = stream(key)
    if s == d:
        rows = np.tile(np.arange(d, dtype=np.int64), (m, 1))
    elif d <= 4 * s * s:
        rows = np.empty((m, s), dtype=np.int64)
        chunk = max(1, 5 * 10**7 // d)
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            keys = rng.random((hi - lo, d))
            rows[lo:hi] = np.argpartition(keys, s - 1, axis=1)[:, :s]
    else:
        rows = rng.integers(0, d, size=(m, s))
        while True:
            srt = np.sort(rows, axis=1)
            bad = np.flatnonzero(np.any(np.diff(srt, axis=1) == 0, axis=1))
            if bad.size == 0:
                break
            rows[bad] = rng.integers(0, d, size=(bad.size, s))
    signs = 2.0 * rng.integers(0, 2, size=(m, s)) - 1.0
    return rows, signs


def sparsesign_map(rows, signs, d: int, m: int) -> scipy.sparse.csr_matrix:
    """sketch.py:111-114."""
    s = rows.shape[1]
    vals = signs.ravel() / math.sqrt(s)
    cols = np.repeat(np.arange(m), s)
    return scipy.sparse.csr_matrix((vals, (rows.ravel(), cols)), shape=(d, m), dtype=np.float64)


def countsketch_map(rows, signs, d: int, m: int) -> scipy.sparse.csr_matrix:
    """sketch.py:100-102."""
    return scipy.sparse.csr_matrix((signs, (rows, np.arange(m))), shape=(d, m), dtype=np.float64)


def countsketch_apply(rows, signs, d: int, A):
    """sketch.py:209-212: `sparse_map @ A` (dense -> csr_matvecs fold; CSR
    operand -> SpGEMM then densify)."""
    m = rows.shape[0]
    smap = countsketch_map(rows, signs, d, m)
    if scipy.sparse.issparse(A):
        return (smap @ scipy.sparse.csr_matrix(A)).toarray()
    return smap @ A


def countsketch_fold(rows, signs, d: int, A: np.ndarray) -> np.ndarray:
    """The same arithmetic as csr_matvecs written out: for every bucket the
    signed rows are added in ascending row order starting from +0.0
    (np.add.at applies updates sequentially in index order)."""
    A2 = A.reshape(A.shape[0], -1)
    out = np.zeros((d, A2.shape[1]))
    np.add.at(out, rows, signs[:, None] * A2)
    return out.reshape((d,) + A.shape[1:])


def fwht_inplace(x: np.ndarray) -> np.ndarray:
    """sketch.py:152-177 (radix-2 passes, h ascending, butterfly
    (a, b) -> (a+b, (a+b) - 2b))."""
    n = x.shape[0]
    work = x.reshape(n, -1)
    h = 1
    while h < n:
        w = work.reshape(n // (2 * h), 2, h, work.shape[1])
        w[:, 0] += w[:, 1]
        w[:, 1] *= -2.0
        w[:, 1] += w[:, 0]
        h *= 2
    return x


def srht_apply(sign_diag, row_sample, m_pad: int, d: int, A: np.ndarray) -> np.ndarray:
    """sketch.py:213-223."""
    arr = A.toarray() if scipy.sparse.issparse(A) else A
    m = arr.shape[0]
    pad_shape = (m_pad,) if arr.ndim == 1 else (m_pad, arr.shape[1])
    pad = np.zeros(pad_shape, dtype=np.float64)
    if arr.ndim == 1:
        pad[:m] = sign_diag[:m] * arr
    else:
        pad[:m] = sign_diag[:m, None] * arr
    fwht_inplace(pad)
    return pad[row_sample] / math.sqrt(d)


def gaussian_apply(G: np.ndarray, A) -> np.ndarray:
    """sketch.py:204-208."""
    if scipy.sparse.issparse(A):
        return np.ascontiguousarray((scipy.sparse.csr_matrix(A).T @ G.T).T)
    return G @ A


# -------------------------------------------------------------- reduced solve
class RankDeficient(Exception):
    def __init__(self, col: int, val: float):
        super().__init__(f"input is numerically rank deficient at column {col} "
                         f"(|R[{col},{col}]| = {val:.3e})")
        self.col, self.val = col, val


def economy_qr(M: np.ndarray):
    """linalg.py:166-192 -> (Q, R) with diag(R) >= 0, or RankDeficient.
    Inputs and outputs are Fortran-ordered like the DenseMatrix carriers."""
    M = np.asfortranarray(M, dtype=np.float64)
    q, r = np.linalg.qr(M, mode="reduced")
    diag = np.diagonal(r).copy()
    flip = diag < 0
    if np.any(flip):
        q = q.copy()
        r = r.copy()
        q[:, flip] *= -1.0
        r[flip, :] *= -1.0
        diag = np.abs(diag)
    fro = float(np.linalg.norm(M))
    bad = np.flatnonzero(diag < RANK_TOL * fro) if fro > 0 else np.arange(M.shape[1])
    if bad.size:
        col = int(bad[0])
        raise RankDeficient(col, float(diag[col]) if fro > 0 else 0.0)
    return np.asfortranarray(q), np.asfortranarray(np.triu(r))


def residual_norm(A, b: np.ndarray, x: np.ndarray) -> float:
    """solvers.py:102-107."""
    return float(np.linalg.norm(A @ x - b))


def sketch_apply(kind: str, key: int, d: int, A, b=None):
    """(SA, Sb) for one operator realisation.  Dense operands are taken in
    Fortran order, as the DenseMatrix carrier stores them (linalg.py:38)."""
    m = A.shape[0]
    if not scipy.sparse.issparse(A):
        A = np.asfortranarray(A, dtype=np.float64)
    if kind == "countsketch":
        rows, signs = countsketch_draws(key, m, d)
        SA = countsketch_apply(rows, signs, d, A)
        Sb = countsketch_apply(rows, signs, d, b) if b is not None else None
    elif kind == "srht":
        sg, rs, m_pad = srht_draws(key, m, d)
        SA = srht_apply(sg, rs, m_pad, d, A)
        Sb = srht_apply(sg, rs, m_pad, d, b) if b is not None else None
    elif kind == "gaussian":
        G = gaussian_draws(key, d, m)
        SA = gaussian_apply(G, A)
        Sb = gaussian_apply(G, b) if b is not None else None
    elif kind == "sparsesign":  # default sparsity s = 8 (sketch.py:52)
        rows, signs = sparsesign_draws(key, m, d, 8)
        smap = sparsesign_map(rows, signs, d, m)
        SA = (smap @ scipy.sparse.csr_matrix(A)).toarray() if scipy.sparse.issparse(A) else smap @ A
        Sb = smap @ b if b is not None else None
    else:
        raise ValueError(kind)
    return SA, Sb


def saa_solve(A, b: np.ndarray, kind: str, seed: int, d_factor: float):
    """solvers.py:296-320 via solve(problem, "saa", SketchSpec(kind, 1, seed),
    SolverOptions(d_factor)) -> dict(x, residual, SA, Sb, d)."""
    m, n = A.shape
    if not scipy.sparse.issparse(A):
        A = np.asfortranarray(A, dtype=np.float64)
    d = default_embed_dim(m, n, d_factor)
    key = operator_key(seed, kind, m, method="saa")
    SA, Sb = sketch_apply(kind, key, d, A, b)
    q, r = economy_qr(SA)
    x = scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False, check_finite=False)
    return {"x": x, "residual": residual_norm(A, b, x), "SA": SA, "Sb": Sb, "d": d, "R": r}


# ------------------------------------------------------------------ SAP / LSQR
_EPS = float(np.finfo(np.float64).eps)  # solvers.py:37


def sym_ortho(a: float, b: float):
    """solvers.py:258-270: stable Givens rotation (c, s, r)."""
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


def lsqr(A, b: np.ndarray, atol: float = 1e-10, btol: float = 1e-10, max_iter=None,
         precond_R=None):
    """solvers.py:110-255 (Paige & Saunders LSQR, optionally right-
    preconditioned by R: operator y -> A R^-1 y, returns x = R^-1 y).
    Returns dict(x, iterations, termination, residual)."""
    n = A.shape[1]
    max_iter = 4 * n if max_iter is None else max_iter
    r = precond_R

    def inv_r(v, transposed=False):
        return scipy.linalg.solve_triangular(r, v, lower=False, trans="T" if transposed else "N",
                                             check_finite=False)

    if r is None:
        mv = lambda v: A @ v  # noqa: E731
        rmv = lambda u: A.T @ u  # noqa: E731
    else:
        mv = lambda v: A @ inv_r(v)  # noqa: E731
        rmv = lambda u: inv_r(A.T @ u, transposed=True)  # noqa: E731
    x = np.zeros(n)
    u = np.array(b, dtype=np.float64, copy=True)
    beta = float(np.linalg.norm(u))
    alfa = 0.0
    v = np.zeros(n)
    if beta > 0:
        u /= beta
        v = rmv(u)
        alfa = float(np.linalg.norm(v))
    if alfa > 0:
        v /= alfa
    w = v.copy()
    itn = istop = 0
    anorm = 0.0
    rhobar, phibar, bnorm = alfa, beta, beta
    if alfa * beta == 0.0:
        xf = x if r is None else inv_r(x)
        return {"x": xf, "iterations": 0, "termination": "atol_btol",
                "residual": residual_norm(A, b, xf)}
    while itn < max_iter:
        itn += 1
        u = mv(v) - alfa * u
        beta = float(np.linalg.norm(u))
        if beta > 0:
            u /= beta
            anorm = math.sqrt(anorm**2 + alfa**2 + beta**2)
            v = rmv(u) - beta * v
            alfa = float(np.linalg.norm(v))
            if alfa > 0:
                v /= alfa
        cs, sn, rho = sym_ortho(rhobar, beta)
        theta = sn * alfa
        rhobar = -cs * alfa
        phi = cs * phibar
        phibar = sn * phibar
        x += (phi / rho) * w
        w = v + (-theta / rho) * w
        rnorm = phibar
        arnorm = alfa * abs(sn * phi)
        xnorm = float(np.linalg.norm(x))
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
    xf = x if r is None else inv_r(x)
    return {"x": xf, "iterations": itn, "termination": "max_iter" if istop == 7 else "atol_btol",
            "residual": residual_norm(A, b, xf)}


def sap_solve(A, b: np.ndarray, kind: str, seed: int, d_factor: float, warm_start: bool = True,
              atol: float = 1e-10, btol: float = 1e-10, max_iter=None):
    """solvers.py:323-361 via solve(problem, "sap", SketchSpec(kind, 1, seed),
    SolverOptions(...)): LSQR right-preconditioned by R of QR(S A), warm
    started from the sketched solution."""
    m, n = A.shape
    if not scipy.sparse.issparse(A):
        A = np.asfortranarray(A, dtype=np.float64)
    d = default_embed_dim(m, n, d_factor)
    key = operator_key(seed, kind, m, method="sap")
    SA, Sb = sketch_apply(kind, key, d, A, b)
    q, r = economy_qr(SA)
    if warm_start:
        x0 = scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False, check_finite=False)
        r0 = b - A @ x0
        inner = lsqr(A, r0, atol, btol, max_iter, precond_R=r)
        x = x0 + inner["x"]
    else:
        inner = lsqr(A, b, atol, btol, max_iter, precond_R=r)
        x = inner["x"]
    return {"x": x, "iterations": inner["iterations"], "termination": inner["termination"],
            "residual": residual_norm(A, b, x), "d": d, "R": r}
