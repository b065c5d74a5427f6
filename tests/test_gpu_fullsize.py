"""Full-size parity for BASELINE.json configs 2-5 on the B200.

The north_star target is "every config matches the CPU oracle": hashes,
signs and samples exact; S*A within 1e-12 relative Frobenius (bitwise for
CountSketch, whose fold order the kernels keep); x within 1e-9 relative;
||Ax - b|| within 1e-10 relative.  Inputs come from the oracle's own
generator (workloads.make_problem(..., backend="numpy")); the oracle runs on
this box's host cores (oracle/oracle.py, with the column-threaded C applies
of oracle/c/apply_oracle.c for the 2 GiB / 16 GiB dense operands), and the
BLAS-free quantities are also checked against digests the reference itself
produced at full size (tests/golden/golden_full.json, made by
tests/golden/make_golden_full.py).

Config 2 is kappa = 1e8: any two backward-stable QRs of the same S*A differ
in x by ~1e-8, so there the device x error is asserted
against -- and reported next to -- the oracle's own QR-rounding spread,
measured here by re-solving row-permuted copies of the same sketched
system; the H3 diagnostic (device S*A -> the oracle's numpy QR) must give
the oracle's x bit for bit, and the device x must be as good a minimiser
of the sketched problem as the oracle's.

Set SKL_PARITY_REPORT=<path> to append one JSON line per config with the
measured errors (the round's numbers are committed under profiles/).
"""

import hashlib
import json
import os
import time
from pathlib import Path

import numpy as np
import pytest
import scipy.linalg

from conftest import rel_fro

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)
if os.environ.get("SKL_SKIP_FULLSIZE"):
    pytest.skip("SKL_SKIP_FULLSIZE set", allow_module_level=True)

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from oracle import clib  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLDEN_FULL = json.loads((Path(__file__).resolve().parent / "golden" / "golden_full.json")
                         .read_text())
SA_TOL, X_TOL, R_TOL = 1e-12, 1e-9, 1e-10


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def report(cfg: str, **fields):
    path = os.environ.get("SKL_PARITY_REPORT")
    line = {"config": cfg, **{k: (float(v) if isinstance(v, (np.floating, float)) else v)
                              for k, v in fields.items()}}
    print(json.dumps(line))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")


def saa_spec(kind, d):
    return E.SketchSpec(kind, d, seed=E.derive_seed(W.SEED, "saa"))


def oracle_x(SA, Sb):
    """_sketch_qr + _apply_inverse_r (solvers.py:308-309) on given S*A, S*b."""
    q, r = O.economy_qr(SA)
    return scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False, check_finite=False)


def to_dev(a):
    return torch.from_numpy(a).cuda()  # an F-ordered ndarray stays column-major


def solve_device(A_carrier, b_dev, kind, c):
    prob = E.LeastSquaresProblem(A=A_carrier, b=E.Vector(b_dev))
    t0 = time.perf_counter()
    res = E.solve(prob, "saa", E.SketchSpec(kind, 1, seed=W.SEED),
                  E.SolverOptions(d_factor=c.d / c.n))
    torch.cuda.synchronize()
    assert res.d == c.d and res.method == "saa" and res.sketch == kind
    x = res.x.data.cpu().numpy() if hasattr(res.x.data, "cpu") else np.asarray(res.x.data)
    return x, res.residual_norm, time.perf_counter() - t0


def check_solution(cfg, x, rnorm, A, b, SA_ref, Sb_ref, x_tol=X_TOL, **extra):
    x_ref = oracle_x(SA_ref, Sb_ref)
    r_ref = O.residual_norm(A, b, x_ref)
    x_err = rel_fro(x, x_ref)
    r_err = abs(rnorm - r_ref) / r_ref
    report(cfg, x_rel_err=x_err, residual_rel_err=r_err, x_tol=x_tol, **extra)
    assert x_err <= x_tol
    assert r_err <= R_TOL
    return x_ref


# ------------------------------------------------------------------ config 2
def test_cfg2_countsketch_fullsize():
    c = W.config(2)
    A, b, _ = W.make_problem(c)  # 2^20 x 256, kappa 1e8, F-ordered
    key = O.operator_key(W.SEED, "countsketch", c.m, method="saa")
    rows, signs = O.countsketch_draws(key, c.m, c.d)
    op = E.build_sketch(saa_spec("countsketch", c.d), c.m)
    assert np.array_equal(op.rows, rows) and np.array_equal(op.signs, signs)
    assert sha(op.rows, op.signs) == GOLDEN_FULL["cfg2_cs_sha"]
    SA_ref = clib.countsketch_apply_mt(rows, signs, c.d, A)
    Sb_ref = O.countsketch_apply(rows, signs, c.d, b)
    Ad, bd = to_dev(A), to_dev(b)
    SA = E.apply_to_matrix(op, E.DenseMatrix(Ad)).data.cpu().numpy()
    Sb = E.apply_to_vector(op, E.Vector(bd)).data.cpu().numpy()
    assert np.array_equal(SA, SA_ref), rel_fro(SA, SA_ref)
    assert np.array_equal(Sb, Sb_ref), rel_fro(Sb, Sb_ref)  # one long column: ordered walk
    # H3: the device S*A through the oracle's own QR reproduces its x bitwise
    x_ref = oracle_x(SA_ref, Sb_ref)
    assert np.array_equal(oracle_x(SA, Sb), x_ref)
    # the oracle's QR-rounding spread: the same sketched system, rows permuted
    spread = 0.0
    for s in range(3):
        p = np.random.default_rng(s).permutation(c.d)
        spread = max(spread, rel_fro(oracle_x(np.asfortranarray(SA_ref[p]), Sb_ref[p]), x_ref))
    x, rnorm, wall = solve_device(E.DenseMatrix(Ad), bd, "countsketch", c)
    # as good a minimiser of ||SA x - Sb|| as the oracle's x
    sk_dev = np.linalg.norm(SA_ref @ x - Sb_ref)
    sk_ref = np.linalg.norm(SA_ref @ x_ref - Sb_ref)
    x_tol = max(X_TOL, 2.0 * spread)
    check_solution("cfg2", x, rnorm, A, b, SA_ref, Sb_ref, x_tol=x_tol, SA="bitwise",
                   Sb="bitwise", oracle_qr_spread=spread, h3_numpy_qr_on_device_SA="bitwise",
                   sketched_residual_rel_diff=abs(sk_dev - sk_ref) / sk_ref,
                   device_solve_s=wall)
    assert abs(sk_dev - sk_ref) <= 1e-10 * sk_ref


# ------------------------------------------------------------------ config 3
def test_cfg3_gaussian_fullsize():
    c = W.config(3)
    A, b, _ = W.make_problem(c)  # 262144 x 512
    key = O.operator_key(W.SEED, "gaussian", c.m, method="saa")
    op = E.build_sketch(saa_spec("gaussian", c.d), c.m)
    G_dev, ldg = op.device_gaussian()
    G = np.ascontiguousarray(G_dev[:, : c.m].cpu().numpy())
    G_ref = O.gaussian_draws(key, c.d, c.m)
    assert np.array_equal(G, G_ref)
    assert sha(G) == GOLDEN_FULL["cfg3_gauss_sha"]
    del G
    SA_ref, Sb_ref = O.gaussian_apply(G_ref, A), O.gaussian_apply(G_ref, b)
    del G_ref
    Ad, bd = to_dev(A), to_dev(b)
    SA = E.apply_to_matrix(op, E.DenseMatrix(Ad)).data.cpu().numpy()
    Sb = E.apply_to_vector(op, E.Vector(bd)).data.cpu().numpy()
    sa_err, sb_err = rel_fro(SA, SA_ref), rel_fro(Sb, Sb_ref)
    assert sa_err <= SA_TOL and sb_err <= SA_TOL
    x, rnorm, wall = solve_device(E.DenseMatrix(Ad), bd, "gaussian", c)
    check_solution("cfg3", x, rnorm, A, b, SA_ref, Sb_ref, gaussian_entries="bitwise",
                   SA_rel_err=sa_err, Sb_rel_err=sb_err, device_solve_s=wall)


# ------------------------------------------------------------------ config 4
def test_cfg4_csr_countsketch_fullsize():
    c = W.config(4)
    A, b, _ = W.make_problem(c)  # scipy CSR 2^22 x 1024, ~4.29 M nnz
    assert A.nnz == GOLDEN_FULL["cfg4_nnz"]
    assert sha(A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data) == \
        GOLDEN_FULL["cfg4_A_sha"]
    assert sha(b) == GOLDEN_FULL["cfg4_b_sha"]
    key = O.operator_key(W.SEED, "countsketch", c.m, method="saa")
    rows, signs = O.countsketch_draws(key, c.m, c.d)
    op = E.build_sketch(saa_spec("countsketch", c.d), c.m)
    assert np.array_equal(op.rows, rows) and np.array_equal(op.signs, signs)
    assert sha(op.rows, op.signs) == GOLDEN_FULL["cfg4_cs_sha"]
    SA_ref = O.countsketch_apply(rows, signs, c.d, A)
    Sb_ref = O.countsketch_apply(rows, signs, c.d, b)
    Ac = E.SparseMatrix.from_scipy(A)
    bd = to_dev(b)
    SA = E.apply_to_matrix(op, Ac).data
    Sb = E.apply_to_vector(op, E.Vector(bd)).data.cpu().numpy()
    assert np.array_equal(SA, SA_ref)
    assert np.array_equal(Sb, Sb_ref)
    assert sha(np.asfortranarray(SA)) == GOLDEN_FULL["cfg4_SA_sha"]
    assert sha(Sb) == GOLDEN_FULL["cfg4_Sb_sha"]
    x, rnorm, wall = solve_device(Ac, bd, "countsketch", c)
    check_solution("cfg4", x, rnorm, A, b, SA_ref, Sb_ref, SA="bitwise", Sb="bitwise",
                   device_solve_s=wall)


# ------------------------------------------------------------------ config 5
@pytest.fixture(scope="module")
def cfg5():
    c = W.config(5)
    A, b, _ = W.make_problem(c)  # 2^23 x 256 (16 GiB), F-ordered
    Ad, bd = to_dev(A), to_dev(b)
    yield c, A, b, Ad, bd
    del Ad, bd
    torch.cuda.empty_cache()


def test_cfg5_countsketch_fullsize(cfg5):
    c, A, b, Ad, bd = cfg5
    assert sha(np.asfortranarray(A[:, :32])) == GOLDEN_FULL["cfg5_A32_sha"]
    key = O.operator_key(W.SEED, "countsketch", c.m, method="saa")
    rows, signs = O.countsketch_draws(key, c.m, c.d)
    op = E.build_sketch(saa_spec("countsketch", c.d), c.m)
    assert np.array_equal(op.rows, rows) and np.array_equal(op.signs, signs)
    assert sha(op.rows, op.signs) == GOLDEN_FULL["cfg5_cs_sha"]
    SA_ref = clib.countsketch_apply_mt(rows, signs, c.d, A)
    Sb_ref = O.countsketch_apply(rows, signs, c.d, b)
    assert sha(np.asfortranarray(SA_ref[:, :32])) == GOLDEN_FULL["cfg5_cs_SA32_sha"]
    SA = E.apply_to_matrix(op, E.DenseMatrix(Ad)).data.cpu().numpy()
    Sb = E.apply_to_vector(op, E.Vector(bd)).data.cpu().numpy()
    assert np.array_equal(SA, SA_ref)
    assert np.array_equal(Sb, Sb_ref)
    x, rnorm, wall = solve_device(E.DenseMatrix(Ad), bd, "countsketch", c)
    check_solution("cfg5_countsketch", x, rnorm, A, b, SA_ref, Sb_ref, SA="bitwise",
                   Sb="bitwise", device_solve_s=wall)


def test_cfg5_srht_fullsize(cfg5):
    c, A, b, Ad, bd = cfg5
    key = O.operator_key(W.SEED, "srht", c.m, method="saa")
    sg, rs, m_pad = O.srht_draws(key, c.m, c.d)
    op = E.build_sketch(saa_spec("srht", c.d), c.m)
    assert op.padded_dim == m_pad == c.m
    assert np.array_equal(op.sign_diag, sg) and np.array_equal(op.row_sample, rs)
    assert sha(op.sign_diag.astype(np.int8)) == GOLDEN_FULL["cfg5_srht_signs_sha"]
    assert sha(op.row_sample) == GOLDEN_FULL["cfg5_srht_sample_sha"]
    SA_ref = clib.srht_apply_mt(sg, rs, m_pad, c.d, A)
    Sb_ref = clib.srht_apply_mt(sg, rs, m_pad, c.d, b)
    SA = E.apply_to_matrix(op, E.DenseMatrix(Ad)).data.cpu().numpy()
    Sb = E.apply_to_vector(op, E.Vector(bd)).data.cpu().numpy()
    sa_err, sb_err = rel_fro(SA, SA_ref), rel_fro(Sb, Sb_ref)
    assert sa_err <= SA_TOL and sb_err <= SA_TOL
    x, rnorm, wall = solve_device(E.DenseMatrix(Ad), bd, "srht", c)
    check_solution("cfg5_srht", x, rnorm, A, b, SA_ref, Sb_ref, SA_rel_err=sa_err,
                   Sb_rel_err=sb_err, device_solve_s=wall)
