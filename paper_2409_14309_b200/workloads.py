"""Seeded synthetic workloads for the five BASELINE.json configs.

No dataset is involved: every array is drawn from a seeded
stream, so the GPU run, the CPU baseline and the parity tests see the same
inputs.  Two generators:

* ``backend="numpy"`` draws from ``stream(derive_seed(seed, tag, cfg))``
  (numpy Philox; reproducible on any box with numpy 2.3.5) -- used by the
  parity tests, the golden fixtures and reduced-size runs;
* ``backend="torch"`` draws the same distributions on the GPU with a
  seeded ``torch.Generator`` -- used for the full-size bench inputs
  (cfg2 needs a 2^20 x 256 QR, cfg5 is 16 GiB), where host generation
  would take minutes.  The values differ from the numpy backend; the
  distributions and shapes do not.

Config shapes (BASELINE.json "configs"):
  1: dense 20000 x 200 N(0,1), CountSketch d=800, noise 1e-3
  2: dense 2^20 x 256 = U diag(logspace(0,-8)) V^T, CountSketch d=2048, noise 1e-6
  3: dense 262144 x 512 N(0,1), Gaussian d=2048, noise 1e-3
  4: CSR 2^22 x 1024, density 1e-3 (Binomial row counts, distinct uniform
     columns, N(0,1) values), CountSketch d=8192, noise 1e-3
  5: dense 2^23 x 256 N(0,1), SRHT d=2048 (and CountSketch d=2048), noise 1e-3
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse

from .rng import derive_seed, stream

SEED = 2409_14309


@dataclass(frozen=True)
class Config:
    cfg: int
    m: int
    n: int
    d: int
    kind: str
    noise: float
    gen: str            # "gauss" | "svd" | "csr"
    kappa: float = 1.0
    density: float = 0.0


CONFIGS = {
    1: Config(1, 20_000, 200, 800, "countsketch", 1e-3, "gauss"),
    2: Config(2, 1 << 20, 256, 2048, "countsketch", 1e-6, "svd", kappa=1e8),
    3: Config(3, 262_144, 512, 2048, "gaussian", 1e-3, "gauss"),
    4: Config(4, 1 << 22, 1024, 8192, "countsketch", 1e-3, "csr", density=1e-3),
    5: Config(5, 1 << 23, 256, 2048, "srht", 1e-3, "gauss"),
}


def config(cfg: int, m: int | None = None, n: int | None = None, d: int | None = None,
           kind: str | None = None) -> Config:
    """A config, optionally with reduced sizes / another sketch kind."""
    c = CONFIGS[cfg]
    return Config(c.cfg, m or c.m, n or c.n, d or c.d, kind or c.kind, c.noise, c.gen, c.kappa,
                  c.density)


def algorithmic_bytes(c: Config, nnz: int | None = None) -> int:
    """Bytes of A and b the sketch must read.
    CSR: 16*nnz + 8*(m+1) (int64 indices + values + indptr) + 8*m for b."""
    if c.gen == "csr":
        return 16 * int(nnz) + 8 * (c.m + 1) + 8 * c.m
    return 8 * c.m * c.n + 8 * c.m


def _csr_numpy(c: Config, seed: int):
    rng = stream(derive_seed(seed, "A", c.cfg))
    m, n = c.m, c.n
    counts = rng.binomial(n, c.density, size=m).astype(np.int64)
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    rowid = np.repeat(np.arange(m, dtype=np.int64), counts)
    cols = rng.integers(0, n, size=nnz)
    # distinct columns per row: redraw the (rare) rows holding a duplicate
    while True:
        order = np.lexsort((cols, rowid))
        cs, rs = cols[order], rowid[order]
        dup = np.flatnonzero((cs[1:] == cs[:-1]) & (rs[1:] == rs[:-1]))
        if dup.size == 0:
            break
        bad_rows = np.unique(rs[dup])
        mask = np.isin(rowid, bad_rows)
        cols[mask] = rng.integers(0, n, size=int(mask.sum()))
    order = np.lexsort((cols, rowid))
    indices = cols[order]
    values = rng.standard_normal(nnz)
    return indptr, indices, values


def make_problem(c: Config, seed: int = SEED, backend: str = "numpy"):
    """(A, b, x_true).  numpy backend: A is an F-ordered ndarray (or a
    scipy CSR for cfg4); torch backend: A is a column-major CUDA tensor
    (or a scipy CSR), b and x_true CUDA tensors."""
    m, n = c.m, c.n
    if c.gen == "csr":
        indptr, indices, values = _csr_numpy(c, seed)
        A = scipy.sparse.csr_matrix((values, indices, indptr), shape=(m, n))
        x = stream(derive_seed(seed, "x", c.cfg)).standard_normal(n)
        noise = stream(derive_seed(seed, "noise", c.cfg)).standard_normal(m)
        b = A @ x + c.noise * noise
        if backend == "torch":
            import torch

            return A, torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda()
        return A, b, x
    if backend == "numpy":
        if c.gen == "svd":
            g = stream(derive_seed(seed, "U", c.cfg)).standard_normal((n, m)).T
            u, _ = np.linalg.qr(g, mode="reduced")
            del g
            v, _ = np.linalg.qr(stream(derive_seed(seed, "V", c.cfg)).standard_normal((n, n)))
            sigma = np.logspace(0.0, -np.log10(c.kappa), n)
            A = np.asfortranarray((u * sigma) @ v.T)
        else:
            A = stream(derive_seed(seed, "A", c.cfg)).standard_normal((n, m)).T
        x = stream(derive_seed(seed, "x", c.cfg)).standard_normal(n)
        noise = stream(derive_seed(seed, "noise", c.cfg)).standard_normal(m)
        b = A @ x + c.noise * noise
        return A, b, x
    import torch

    gen = torch.Generator(device="cuda")
    gen.manual_seed(derive_seed(seed, "A", c.cfg) & ((1 << 63) - 1))
    f64 = torch.float64
    if c.gen == "svd":
        g = torch.randn((n, m), generator=gen, device="cuda", dtype=f64).t()
        u, _ = torch.linalg.qr(g, mode="reduced")
        del g
        vg = torch.randn((n, n), generator=gen, device="cuda", dtype=f64)
        v, _ = torch.linalg.qr(vg)
        sigma = torch.logspace(0.0, -float(np.log10(c.kappa)), n, dtype=f64, device="cuda")
        A = ((u * sigma) @ v.t())
        del u
        A = A.t().contiguous().t()
    else:
        A = torch.randn((n, m), generator=gen, device="cuda", dtype=f64).t()
    x = torch.randn((n,), generator=gen, device="cuda", dtype=f64)
    noise = torch.randn((m,), generator=gen, device="cuda", dtype=f64)
    b = A @ x + c.noise * noise
    return A, b, x
