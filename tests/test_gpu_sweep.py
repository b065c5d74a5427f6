"""Seeded random sweep of the public apply API against the oracle: every
sketch kind, dense host / dense device / CSR operands, ragged shapes
(m, n, d not multiples of anything, d > n, d close to m), vectors too.
CountSketch and sparse sign are bitwise; SRHT and Gaussian within 1e-13."""

import numpy as np
import pytest
import scipy.sparse

from conftest import rel_fro

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_14309_b200 as E  # noqa: E402
from oracle import oracle as O  # noqa: E402

KINDS = ("countsketch", "sparsesign", "srht", "gaussian")


def _case(i: int):
    rng = np.random.default_rng(1000 + i)
    kind = KINDS[i % 4]
    layout = ("host", "device", "csr")[(i // 4) % 3]
    m = int(rng.integers(1, 30000))
    n = int(rng.integers(1, 24))
    dmax = min(m, 2048 if kind in ("countsketch", "sparsesign") else 1024)
    if kind == "gaussian":
        dmax = min(dmax, max(1, 4_000_000 // m))
    d = int(rng.integers(1, dmax + 1))
    return rng, kind, layout, m, n, d


@pytest.mark.parametrize("i", range(72))
def test_random_shapes_match_oracle(i):
    rng, kind, layout, m, n, d = _case(i)
    seed = int(rng.integers(0, 2**31))
    if layout == "csr":
        A = scipy.sparse.random(m, n, density=float(rng.uniform(0.0, 0.3)), random_state=i,
                                format="csr")
        A.data = rng.standard_normal(A.nnz)
        carrier = E.SparseMatrix.from_scipy(A)
    else:
        A = rng.standard_normal((m, n))
        if layout == "device":
            carrier = E.DenseMatrix(torch.from_numpy(np.asfortranarray(A)).cuda())
        else:
            carrier = E.DenseMatrix(A)
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec(kind, d, seed=seed), m)
    SA = E.apply_to_matrix(op, carrier).to_numpy()
    Sb = E.apply_to_vector(op, E.Vector(b)).to_numpy()
    want_A, want_b = O.sketch_apply(kind, O.operator_key(seed, kind, m), d, A, b)
    want_A = np.asarray(want_A)
    assert SA.shape == (d, n) and Sb.shape == (d,)
    if kind in ("countsketch", "sparsesign"):
        assert np.array_equal(SA, want_A), (kind, layout, m, n, d)
        assert np.array_equal(Sb, want_b), (kind, layout, m, n, d)
    else:
        assert rel_fro(SA, want_A) <= 1e-13, (kind, layout, m, n, d)
        assert rel_fro(Sb, want_b) <= 1e-13, (kind, layout, m, n, d)


@pytest.mark.parametrize("i", range(16))
def test_random_saa_solves_match_oracle(i):
    """solve(problem, "saa", spec, opts) on random well-conditioned shapes:
    x within 1e-9 and the residual within 1e-10 of the oracle's."""
    rng = np.random.default_rng(5000 + i)
    kind = KINDS[i % 4]
    n = int(rng.integers(1, 40))
    m = int(rng.integers(4 * n + 1, 20000))
    d_factor = float(rng.uniform(2.0, 6.0))
    A = rng.standard_normal((m, n))
    b = A @ rng.standard_normal(n) + 1e-3 * rng.standard_normal(m)
    seed = int(rng.integers(0, 2**31))
    want = O.saa_solve(A, b, kind, seed, d_factor)
    res = E.solve(E.LeastSquaresProblem(A=E.DenseMatrix(A), b=E.Vector(b)), "saa",
                  E.SketchSpec(kind, 1, seed=seed), E.SolverOptions(d_factor=d_factor))
    assert res.d == want["d"]
    assert rel_fro(res.x.data, want["x"]) <= 1e-9, (kind, m, n, res.d)
    assert abs(res.residual_norm - want["residual"]) <= 1e-10 * want["residual"]


@pytest.mark.parametrize("i", range(12))
def test_random_sap_lsqr_direct_match_oracle(i):
    """sap (all kinds, warm start on/off, dense and CSR), plain lsqr and
    direct on random shapes: x within 1e-9 of the oracle / LAPACK."""
    rng = np.random.default_rng(7000 + i)
    n = int(rng.integers(2, 30))
    m = int(rng.integers(6 * n, 15000))
    A = rng.standard_normal((m, n)) * np.logspace(0, -3, n)
    if i % 3 == 2:
        S = scipy.sparse.random(m, n, density=0.2, random_state=i, format="csr")
        S.data = rng.standard_normal(S.nnz)
        A = S.toarray() + np.eye(m, n)  # full column rank
        carrier = E.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(A))
    else:
        carrier = E.DenseMatrix(A)
    b = A @ rng.standard_normal(n) + 1e-2 * rng.standard_normal(m)
    prob = E.LeastSquaresProblem(A=carrier, b=E.Vector(b))
    kind = KINDS[i % 4]
    seed = int(rng.integers(0, 2**31))
    warm = bool(i % 2)
    want = O.sap_solve(A, b, kind, seed, 4.0, warm_start=warm)
    res = E.solve(prob, "sap", E.SketchSpec(kind, 1, seed=seed),
                  E.SolverOptions(d_factor=4.0, warm_start=warm))
    assert res.iterations == want["iterations"], (kind, m, n)
    assert rel_fro(res.x.data, want["x"]) <= 1e-9, (kind, m, n)
    # unpreconditioned LSQR on kappa ~1e3..1e4: the iterates amplify the
    # different rounding of the device reductions; compare to that bound
    plain = E.solve(prob, "lsqr")
    ref = O.lsqr(A, b)
    assert rel_fro(plain.x.data, ref["x"]) <= 1e-7
    assert abs(plain.residual_norm - ref["residual"]) <= 1e-10 * ref["residual"]
    assert abs(plain.iterations - ref["iterations"]) <= max(2, ref["iterations"] // 10)
    direct = E.solve(prob, "direct")
    assert rel_fro(direct.x.data, np.linalg.lstsq(A, b, rcond=None)[0]) <= 1e-10
