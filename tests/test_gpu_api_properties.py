"""The reference package's public-API properties, checked on the device engine.

These restate, against `paper_2409_14309_b200`, the behaviours the reference
asserts of its own `sketchls` API: apply-vs-materialisation, sparse-vs-dense
operands, vector-vs-single-column, linearity, isometry in expectation and the
subspace embedding (/root/reference/pkg/tests/test_sketch.py:139-248), and the
solver contracts of SAA / SAP / the dispatcher
(/root/reference/pkg/tests/test_solvers.py:99-230).  Sizes and seeds are this
suite's own; every apply runs through the native library.  Needs a B200.
"""

import numpy as np
import pytest
import scipy.sparse

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200.rng import derive_seed, stream  # noqa: E402

ALL_KINDS = ("gaussian", "srht", "countsketch", "sparsesign", "identity")
SKETCH_KINDS = ("gaussian", "srht", "countsketch", "sparsesign")


def host(a):
    """Carrier payloads as ndarrays (generate_problem keeps its problems on the
    device, so their solutions come back as device tensors)."""
    return a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a, dtype=np.float64)


def rel_err(x, y):
    x, y = host(x), host(y)
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


# LSQR iteration counts the reference reports on this suite's instances
# (sketchls imported from /root/reference in the build container, same
# ProblemSpec / SketchSpec seeds; the reference tree does not travel to the
# GPU box, so the counts are pinned here).
REF_ITERS = {"sap_well": 12, "sap_ill": 24, "sap_identity": 1, "sap_cold": 34,
             "dispatch_lsqr": 32, "dispatch_sap": 14}


def dense_problem(seed, m, n):
    rng = stream(seed)
    return E.LeastSquaresProblem(A=E.DenseMatrix(rng.standard_normal((m, n))),
                                 b=E.Vector(rng.standard_normal(m)))


# ------------------------------------------------------------------ operators


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_apply_equals_materialised_product(kind):
    m, d, n = 96, 24, 7
    op = E.build_sketch(E.SketchSpec(kind, d, seed=501), m=m)
    a = stream(502).standard_normal((m, n))
    got = E.apply_to_matrix(op, E.DenseMatrix(a)).data
    want = E.materialize(op).data @ a
    assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1.0)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_csr_operand_equals_dense_operand(kind):
    rng = stream(503)
    a = np.where(rng.random((96, 9)) < 0.25, rng.standard_normal((96, 9)), 0.0)
    op = E.build_sketch(E.SketchSpec(kind, 24, seed=504), m=96)
    got = E.apply_to_matrix(op, E.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(a))).data
    want = E.apply_to_matrix(op, E.DenseMatrix(a)).data
    assert np.allclose(got, want, rtol=1e-13, atol=1e-300)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_vector_apply_equals_one_column_matrix(kind):
    m = 80
    op = E.build_sketch(E.SketchSpec(kind, 20, seed=505), m=m)
    b = stream(506).standard_normal(m)
    via_vec = E.apply_to_vector(op, E.Vector(b)).data
    via_mat = E.apply_to_matrix(op, E.DenseMatrix(b.reshape(-1, 1))).data[:, 0]
    assert np.allclose(via_vec, via_mat, rtol=1e-15, atol=1e-300)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_apply_is_linear(kind):
    m = 160
    op = E.build_sketch(E.SketchSpec(kind, 40, seed=507), m=m)
    rng = stream(508)
    u, v = rng.standard_normal(m), rng.standard_normal(m)
    lhs = E.apply_to_vector(op, E.Vector(-1.5 * u + 4 * v)).data
    rhs = (-1.5 * E.apply_to_vector(op, E.Vector(u)).data
           + 4 * E.apply_to_vector(op, E.Vector(v)).data)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_operator_build_is_deterministic(kind):
    spec = E.SketchSpec(kind, 16, seed=509)
    E.clear_operator_cache()
    a = E.materialize(E.build_sketch(spec, m=72)).data
    E.clear_operator_cache()
    b = E.materialize(E.build_sketch(spec, m=72)).data
    assert np.array_equal(a, b)


def test_zero_operand_sketches_to_exact_zero():
    for kind in SKETCH_KINDS:
        op = E.build_sketch(E.SketchSpec(kind, 8, seed=510), m=40)
        out = E.apply_to_matrix(op, E.DenseMatrix(np.zeros((40, 3)))).data
        assert np.array_equal(out, np.zeros((8, 3))), kind


def test_identity_operator_is_exact():
    a = stream(511).standard_normal((15, 4))
    op = E.build_sketch(E.SketchSpec("identity", 15), m=15)
    assert np.array_equal(E.apply_to_matrix(op, E.DenseMatrix(a)).data, a)
    b = stream(512).standard_normal(15)
    assert np.array_equal(E.apply_to_vector(op, E.Vector(b)).data, b)


def test_row_count_mismatch_raises_shape_error():
    op = E.build_sketch(E.SketchSpec("countsketch", 4, seed=0), m=12)
    with pytest.raises(E.ShapeError):
        E.apply_to_matrix(op, E.DenseMatrix(np.ones((13, 2))))
    with pytest.raises(E.ShapeError):
        E.apply_to_vector(op, E.Vector(np.ones(11)))


def test_materialize_guard_raises_capacity_error():
    op = E.build_sketch(E.SketchSpec("countsketch", 2500, seed=0), m=5000)
    with pytest.raises(E.CapacityError):
        E.materialize(op)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_norm_preserved_in_expectation(kind):
    m, d, trials = 1024, 256, 120
    total = 0.0
    for t in range(trials):
        u = stream(derive_seed(3100, kind, t)).standard_normal(m)
        u /= np.linalg.norm(u)
        op = E.build_sketch(E.SketchSpec(kind, d, seed=derive_seed(3200, kind, t)), m=m)
        total += float(np.linalg.norm(E.apply_to_vector(op, E.Vector(u)).data) ** 2)
    assert 0.88 <= total / trials <= 1.12


def test_countsketch_is_a_subspace_embedding():
    m, n = 5000, 40
    basis, _ = np.linalg.qr(stream(513).standard_normal((m, n)))
    op = E.build_sketch(E.SketchSpec("countsketch", 4 * n, seed=514), m=m)
    sa = E.apply_to_matrix(op, E.DenseMatrix(basis)).data
    rng = stream(515)
    good = 0
    for _ in range(100):
        x = rng.standard_normal(n)
        good += 0.5 <= np.linalg.norm(sa @ x) / np.linalg.norm(basis @ x) <= 1.5
    assert good >= 99


def test_gaussian_operator_entry_statistics():
    m, d = 400, 50
    mat = E.materialize(E.build_sketch(E.SketchSpec("gaussian", d, seed=516), m=m)).data
    assert abs(mat.mean()) <= 3 * (1 / np.sqrt(d)) / np.sqrt(d * m)
    assert np.std(mat) == pytest.approx(1 / np.sqrt(d), rel=0.05)


# -------------------------------------------------------------------- solvers


def test_identity_sketch_saa_equals_direct_qr():
    prob = dense_problem(520, 120, 15)
    ref = E.normal_equations_oracle(prob.A, prob.b)
    res = E.sketch_and_apply(prob, E.SketchSpec("identity", 1))
    assert rel_err(res.x.data, ref.data) <= 1e-12
    assert res.iterations == 0 and res.method == "saa"


@pytest.mark.parametrize("kind", SKETCH_KINDS)
def test_consistent_system_recovered_by_saa(kind):
    prob = E.generate_problem(E.ProblemSpec(m=500, n=25, kappa=1e3, beta=0.0, seed=521))
    res = E.sketch_and_apply(prob, E.SketchSpec(kind, 1, seed=522))
    assert rel_err(res.x.data, prob.x_star.data) <= 1e-10 * 1e3


def test_saa_residual_within_twice_optimum():
    prob = dense_problem(523, 600, 25)
    ref = E.normal_equations_oracle(prob.A, prob.b)
    best = np.linalg.norm(prob.A.data @ ref.data - prob.b.data)
    res = E.sketch_and_apply(prob, E.SketchSpec("countsketch", 1, seed=524))
    assert res.d == 100
    assert res.residual_norm <= 2 * best


def test_saa_rank_deficiency_carries_sketch_context():
    rng = stream(525)
    a = rng.standard_normal((60, 5))
    a[:, 4] = a[:, 1]
    prob = E.LeastSquaresProblem(A=E.DenseMatrix(a), b=E.Vector(rng.standard_normal(60)))
    with pytest.raises(E.SingularFactorError, match="countsketch.*d=20"):
        E.sketch_and_apply(prob, E.SketchSpec("countsketch", 1, seed=526))


def test_saa_on_tall_noisy_problem():
    prob = E.generate_problem(E.ProblemSpec(m=40_000, n=80, kappa=1e4, beta=1e-8, seed=527))
    res = E.sketch_and_apply(prob, E.SketchSpec("countsketch", 1, seed=528))
    assert res.d == 320
    assert res.residual_norm <= 2 * prob.beta + 1e-12


def test_sap_well_conditioned_converges_fast():
    prob = E.generate_problem(E.ProblemSpec(m=300, n=12, kappa=10.0, beta=1e-6, seed=530))
    res = E.sketch_and_precondition(prob, E.SketchSpec("countsketch", 1, seed=531))
    assert res.termination == "atol_btol"
    assert res.iterations == REF_ITERS["sap_well"] <= 12


def test_sap_ill_conditioned_forward_error():
    prob = E.generate_problem(E.ProblemSpec(m=6000, n=60, kappa=1e6, beta=1e-10, seed=532))
    res = E.sketch_and_precondition(prob, E.SketchSpec("countsketch", 1, seed=533))
    assert rel_err(res.x.data, prob.x_star.data) <= 1e-8
    assert res.iterations == REF_ITERS["sap_ill"]


def test_sap_identity_sketch_is_an_exact_preconditioner():
    prob = E.generate_problem(E.ProblemSpec(m=150, n=9, kappa=1e2, beta=1e-8, seed=534))
    res = E.sketch_and_precondition(prob, E.SketchSpec("identity", 1, seed=535))
    assert res.iterations == REF_ITERS["sap_identity"] <= 3
    assert rel_err(res.x.data, prob.x_star.data) <= 1e-10


def test_sap_cold_start_converges():
    prob = E.generate_problem(E.ProblemSpec(m=2500, n=30, kappa=1e4, beta=1e-8, seed=536))
    res = E.sketch_and_precondition(prob, E.SketchSpec("countsketch", 1, seed=537),
                                    E.SolverOptions(warm_start=False))
    assert res.termination == "atol_btol"
    assert rel_err(res.x.data, prob.x_star.data) <= 1e-6
    # this problem stops right at the atol/btol boundary (final residual
    # 1e-8 = beta): generate_problem's device QR rounds differently from the
    # reference's numpy QR, so the reference's count is pinned to within one
    # iteration, and the oracle run on this very (device-generated) problem
    # must stop within one iteration of the device run
    assert abs(res.iterations - REF_ITERS["sap_cold"]) <= 1
    from oracle import oracle as O

    A_h, b_h = host(prob.A.data), host(prob.b.data)
    want = O.sap_solve(A_h, b_h, "countsketch", 537, 4.0, warm_start=False)
    assert want["termination"] == "atol_btol"
    assert abs(res.iterations - want["iterations"]) <= 1


def test_sap_csr_operand_matches_dense():
    rng = stream(538)
    a = np.where(rng.random((320, 14)) < 0.4, rng.standard_normal((320, 14)), 0.0)
    b = rng.standard_normal(320)
    spec = E.SketchSpec("countsketch", 1, seed=539)
    dres = E.sketch_and_precondition(E.LeastSquaresProblem(A=E.DenseMatrix(a), b=E.Vector(b)), spec)
    sres = E.sketch_and_precondition(
        E.LeastSquaresProblem(A=E.SparseMatrix.from_scipy(scipy.sparse.csr_matrix(a)),
                              b=E.Vector(b)), spec)
    assert rel_err(sres.x.data, dres.x.data) <= 1e-9


@pytest.mark.parametrize("method", ["lsqr", "saa", "sap"])
def test_dispatcher_is_transparent(method):
    prob = E.generate_problem(E.ProblemSpec(m=350, n=14, kappa=1e3, beta=1e-6, seed=540))
    spec = E.SketchSpec("countsketch", 1, seed=541)
    opts = E.SolverOptions()
    via_solve = E.solve(prob, method, spec, opts)
    direct = {
        "lsqr": lambda: E.lsqr(prob.A, prob.b, opts),
        "saa": lambda: E.sketch_and_apply(prob, spec, opts),
        "sap": lambda: E.sketch_and_precondition(prob, spec, opts),
    }[method]()
    assert np.array_equal(host(via_solve.x.data), host(direct.x.data))
    assert via_solve.iterations == direct.iterations
    if method == "sap":
        assert via_solve.iterations == REF_ITERS["dispatch_sap"]
    elif method == "lsqr":
        # unpreconditioned (kappa 1e3): generate_problem's device QR rounds
        # differently from numpy's, which may move the stopping test by one
        assert abs(via_solve.iterations - REF_ITERS["dispatch_lsqr"]) <= 1


def test_direct_method_equals_qr_oracle_bitwise():
    prob = dense_problem(542, 110, 18)
    ref = E.normal_equations_oracle(prob.A, prob.b)
    res = E.solve(prob, "direct")
    assert np.array_equal(res.x.data, ref.data)
    assert res.termination == "direct"


def test_dispatcher_rejects_bad_requests():
    with pytest.raises(E.SpecError):
        E.solve(dense_problem(543, 30, 3), "cg")
    rng = stream(544)
    wide = E.LeastSquaresProblem(A=E.DenseMatrix(rng.standard_normal((3, 6))),
                                 b=E.Vector(rng.standard_normal(3)))
    with pytest.raises(E.ShapeError):
        E.solve(wide, "saa")
    assert E.solve(dense_problem(545, 40, 4), "lsqr").wall_time_s > 0


def test_solve_many_equals_solve_bitwise():
    """solve_many (two streams, one host sync) returns, for every problem,
    exactly what solve() returns for it alone -- dense device, dense host and
    CSR operands, several sketch kinds, repeated problems."""
    probs = [E.generate_problem(E.ProblemSpec(m=3000 + 100 * i, n=20 + i, kappa=10.0 ** (i % 4),
                                              beta=1e-6, seed=700 + i)) for i in range(5)]
    rng = np.random.default_rng(3)
    csr = scipy.sparse.random(4000, 40, density=0.05, random_state=rng, format="csr")
    probs.append(E.LeastSquaresProblem(E.SparseMatrix.from_scipy(csr), E.Vector(rng.standard_normal(4000))))
    dense_h = rng.standard_normal((2500, 30))
    probs.append(E.LeastSquaresProblem(E.DenseMatrix(np.asfortranarray(dense_h)),
                                       E.Vector(dense_h @ rng.standard_normal(30))))
    probs.append(probs[0])
    for kind in ("countsketch", "srht", "gaussian"):
        spec = E.SketchSpec(kind, 1, seed=11)
        many = E.solve_many(probs, "saa", spec)
        for p, r in zip(probs, many):
            one = E.solve(p, "saa", spec)
            assert np.array_equal(host(r.x.data), host(one.x.data))
            assert r.residual_norm == one.residual_norm
            assert r.d == one.d and r.method == "saa"
