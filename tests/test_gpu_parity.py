"""GPU parity: the CUDA engine (through the C-ABI) against the oracle and the
reference-generated golden fixtures.  Needs a B200."""

import hashlib

import numpy as np
import pytest
import scipy.sparse

from conftest import rel_fro

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native  # noqa: E402
from paper_2409_14309_b200 import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def saa_op(c, kind):
    spec = E.SketchSpec(kind, c.d, seed=E.derive_seed(W.SEED, "saa"))
    return E.build_sketch(spec, c.m)


_LIVE = {}


def live_case(name, golden_meta):
    """Inputs regenerated on this box plus the oracle's results on them.

    b = A @ x (and cfg2's U diag(s) V^T) go through the host BLAS, whose
    rounding depends on the CPU, so parity is checked against the oracle run
    live on the same inputs; the oracle itself is pinned to the reference's
    golden vectors by tests/test_oracle_golden.py."""
    if name not in _LIVE:
        m, n, d = golden_meta[f"{name}_shape"]
        cfg = int(name[3])
        kind = "countsketch" if name.endswith("_cs") else W.CONFIGS[cfg].kind
        c = W.config(cfg, m=m, n=n, d=d)
        A, b, _ = W.make_problem(c)
        _LIVE[name] = (c, kind, A, b, O.saa_solve(A, b, kind, W.SEED, d / n))
    return _LIVE[name]


# ----------------------------------------------------------- CountSketch dense
def test_countsketch_cfg1_bitwise(golden, golden_meta):
    c, _, A, b, ref = live_case("cfg1", golden_meta)
    op = saa_op(c, "countsketch")
    SA = E.apply_to_matrix(op, E.DenseMatrix(A)).data
    Sb = E.apply_to_vector(op, E.Vector(b)).data
    assert np.array_equal(SA, golden["cfg1_SA"])  # A is BLAS-free: golden applies
    assert np.array_equal(SA, ref["SA"])
    assert np.array_equal(Sb, ref["Sb"])


def test_countsketch_device_carriers_bitwise(golden):
    c = W.config(1)
    A, b, _ = W.make_problem(c)
    op = saa_op(c, "countsketch")
    SA = E.apply_to_matrix(op, E.DenseMatrix(torch.from_numpy(A).cuda())).data
    assert SA.is_cuda
    assert np.array_equal(SA.cpu().numpy(), golden["cfg1_SA"])


@pytest.mark.parametrize("name", ["cfg2r", "cfg4r", "cfg5r_cs"])
def test_countsketch_reduced_configs_bitwise(golden, golden_meta, name):
    c, _, A, b, ref = live_case(name, golden_meta)
    sparse = scipy.sparse.issparse(A)
    Ad = A.toarray() if sparse else A  # dense kernel on the same values
    op = saa_op(c, "countsketch")
    SA = E.apply_to_matrix(op, E.DenseMatrix(Ad)).data
    assert np.array_equal(SA, ref["SA"])
    assert np.array_equal(E.apply_to_vector(op, E.Vector(b)).data, ref["Sb"])
    if sparse:  # BLAS-free inputs: the reference's own digest applies too
        assert sha(np.asfortranarray(SA)) == golden_meta[f"{name}_SA_sha"]
        SAc = E.apply_to_matrix(op, E.SparseMatrix.from_scipy(A)).data
        assert np.array_equal(SAc, ref["SA"])


@pytest.mark.parametrize("m,n,d", [(1, 1, 1), (7, 3, 2), (33, 5, 7), (2048, 1, 2048),
                                   (5000, 9, 4096), (12_345, 17, 800), (4099, 260, 300)])
def test_countsketch_ragged_shapes(m, n, d):
    rng = np.random.default_rng(m * 31 + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=m + d), m)
    key = O.derive_seed(m + d, "countsketch", m)
    rows, signs = O.countsketch_draws(key, m, d)
    assert np.array_equal(op.rows, rows) and np.array_equal(op.signs, signs)
    want = O.countsketch_apply(rows, signs, d, A)
    assert np.array_equal(E.apply_to_matrix(op, E.DenseMatrix(A)).data, want)


def test_countsketch_partitions_deterministic():
    """The row-partitioned column kernel (few columns on a long source, used
    beyond the ordered walk's 64 MiB column bound): deterministic, <= 1e-15."""
    m, n, d = 300_000, 3, 2048
    rng = np.random.default_rng(3)
    A = torch.from_numpy(np.asfortranarray(rng.standard_normal((m, n)))).cuda()
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=9), m)
    plan = op.device_plan()
    outs = []
    for _ in range(2):
        SA = torch.empty((n, d), dtype=torch.float64, device="cuda").t()
        plan.apply(A, m, n, m, None, SA, d, None, partitions=0)  # auto: P > 1 here
        outs.append(SA.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    want = O.countsketch_apply(op.rows.astype(np.int64), op.signs.astype(np.float64), d,
                               A.cpu().numpy())
    assert rel_fro(outs[0], want) <= 1e-15


@pytest.mark.parametrize("m,n,d,kind", [(300_000, 3, 2048, "countsketch"),
                                        (1 << 20, 0, 2048, "countsketch"),
                                        (1 << 22, 0, 8192, "countsketch"),
                                        (262_145, 1, 5000, "countsketch"),
                                        (400_000, 2, 1000, "sparsesign")])
def test_countsketch_few_long_columns_bitwise(m, n, d, kind):
    """Few columns on a long source (a vector S b, cfg4's Sb): the ordered
    bucket walk keeps scipy's per-bucket fold, so the result is bitwise."""
    rng = np.random.default_rng(m + n)
    op = E.build_sketch(E.SketchSpec(kind, d, seed=m ^ d, sparsity=4), m)
    smap = op.sparse_map
    if n == 0:
        v = rng.standard_normal(m)
        got = E.apply_to_vector(op, E.Vector(torch.from_numpy(v).cuda())).data.cpu().numpy()
        assert np.array_equal(got, smap @ v)
        return
    A = np.asfortranarray(rng.standard_normal((m, n)))
    got = E.apply_to_matrix(op, E.DenseMatrix(torch.from_numpy(A).cuda())).data.cpu().numpy()
    assert np.array_equal(got, smap @ A)
    b = rng.standard_normal(m)
    from paper_2409_14309_b200.sketch import _countsketch_dense_device

    SA, Sb = _countsketch_dense_device(op, torch.from_numpy(A).cuda(), m, n,
                                       b=torch.from_numpy(b).cuda())
    assert np.array_equal(SA.cpu().numpy(), smap @ A)
    assert np.array_equal(Sb.cpu().numpy(), smap @ b)


def test_countsketch_misaligned_device_view():
    m, n, d = 4001, 4, 64
    base = torch.randn((m + 1, n), dtype=torch.float64, device="cuda").t().contiguous().t()
    view = base[1:, :]  # odd offset, ld = m+1
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=1), m)
    got = E.apply_to_matrix(op, E.DenseMatrix(view)).data.cpu().numpy()
    want = O.countsketch_apply(op.rows.astype(np.int64), op.signs.astype(np.float64), d,
                               view.cpu().numpy())
    assert np.array_equal(got, want)


def test_countsketch_zero_and_linearity():
    m, n, d = 10_000, 6, 512
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=4), m)
    Z = E.apply_to_matrix(op, E.DenseMatrix(np.zeros((m, n)))).data
    assert np.array_equal(Z, np.zeros((d, n)))
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(m), rng.standard_normal(m)
    lhs = E.apply_to_vector(op, E.Vector(2 * u + 3 * v)).data
    rhs = 2 * E.apply_to_vector(op, E.Vector(u)).data + 3 * E.apply_to_vector(op, E.Vector(v)).data
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_shape_errors():
    op = E.build_sketch(E.SketchSpec("countsketch", 4, seed=0), 10)
    with pytest.raises(E.ShapeError):
        E.apply_to_matrix(op, E.DenseMatrix(np.ones((11, 2))))
    with pytest.raises(E.ShapeError):
        E.apply_to_vector(op, E.Vector(np.ones(9)))


# ------------------------------------------------------------------- QR / SAA
@pytest.mark.parametrize("m,n", [(5, 3), (20, 5), (100, 40)])
def test_economy_qr_matches_reference(golden, m, n):
    f = E.economy_qr(E.DenseMatrix(golden[f"qr_M_{m}_{n}"]))
    Q, R = f.Q.data, f.R.data
    assert np.all(np.diagonal(R) >= 0)
    assert np.array_equal(np.tril(R, -1), np.zeros((n, n)))
    assert rel_fro(R, golden[f"qr_R_{m}_{n}"]) <= 1e-13
    assert rel_fro(Q, golden[f"qr_Q_{m}_{n}"]) <= 1e-12


def test_economy_qr_rank_deficiency_names_column():
    a = np.random.default_rng(3).standard_normal((10, 3))
    a[:, 2] = a[:, 1]
    with pytest.raises(E.SingularFactorError, match="column 2"):
        E.economy_qr(E.DenseMatrix(a))


def test_economy_qr_wide_rejected():
    with pytest.raises(E.ShapeError):
        E.economy_qr(E.DenseMatrix(np.array([[1.0, 2.0, 3.0]])))


@pytest.mark.parametrize("name,x_tol", [("cfg1", 1e-9), ("cfg2r", 5e-8), ("cfg4r", 1e-9),
                                        ("cfg5r_cs", 1e-9)])
def test_saa_countsketch_matches_reference(golden, golden_meta, name, x_tol):
    # cfg2 is kappa=1e8: QR rounding alone moves x by ~1e-8
    c, kind, A, b, ref = live_case(name, golden_meta)
    Ac = E.SparseMatrix.from_scipy(A) if scipy.sparse.issparse(A) else E.DenseMatrix(A)
    prob = E.LeastSquaresProblem(A=Ac, b=E.Vector(b))
    res = E.solve(prob, "saa", E.SketchSpec("countsketch", 1, seed=W.SEED),
                  E.SolverOptions(d_factor=c.d / c.n))
    assert res.d == c.d and res.method == "saa" and res.termination == "direct"
    err = rel_fro(res.x.data, ref["x"])
    assert err <= x_tol, f"x vs live oracle: {err:.3e} > {x_tol:.1e}"
    rerr = abs(res.residual_norm - ref["residual"]) / ref["residual"]
    assert rerr <= 1e-10, f"residual vs live oracle: {rerr:.3e}"
    # and against the reference's own numbers from the build box
    gerr = rel_fro(res.x.data, golden[f"{name}_x"])
    assert gerr <= x_tol, f"x vs golden: {gerr:.3e} > {x_tol:.1e} (live oracle: {err:.3e})"
    ref_r = golden_meta[f"{name}_residual"]
    assert abs(res.residual_norm - ref_r) <= 1e-10 * ref_r


def test_saa_rank_deficient_message(golden):
    a, b = golden["rankdef_A"], golden["rankdef_b"]
    prob = E.LeastSquaresProblem(A=E.DenseMatrix(a), b=E.Vector(b))
    with pytest.raises(E.SingularFactorError, match="countsketch.*d=16"):
        E.sketch_and_apply(prob, E.SketchSpec("countsketch", 1, seed=16))


def test_saa_identity_equals_direct_qr():
    rng = np.random.default_rng(10)
    a, b = rng.standard_normal((100, 20)), rng.standard_normal(100)
    res = E.sketch_and_apply(E.LeastSquaresProblem(E.DenseMatrix(a), E.Vector(b)),
                             E.SketchSpec("identity", 1))
    want = np.linalg.lstsq(a, b, rcond=None)[0]
    assert rel_fro(res.x.data, want) <= 1e-12


def test_residual_kernel():
    rng = np.random.default_rng(5)
    m, n = 100_001, 37
    a = np.asfortranarray(rng.standard_normal((m, n)))
    x, b = rng.standard_normal(n), rng.standard_normal(m)
    from paper_2409_14309_b200.solvers import _residual_device

    ta = torch.from_numpy(a).cuda()
    got = _residual_device(E.DenseMatrix(ta), ta, m, torch.from_numpy(b).cuda(),
                           torch.from_numpy(x).cuda())
    want = np.linalg.norm(a @ x - b)
    assert abs(got - want) <= 1e-12 * want


@pytest.mark.parametrize("kind", ["owned", "lanes"])
def test_host_streaming_abi_bitwise(golden, golden_meta, kind):
    """skl_countsketch_dense{_owned}_host: host buffers in/out, H2D streamed."""
    from paper_2409_14309_b200.sketch import CountSketchPlan

    c, _, A, b, ref = live_case("cfg1", golden_meta)
    A = np.asfortranarray(A)
    op = saa_op(c, "countsketch")
    plan = CountSketchPlan(op.rows, op.signs, c.d, kind=kind)
    SA = np.empty((c.d, c.n), order="F")
    Sb = np.empty(c.d)
    plan.apply_host(A, c.m, c.n, c.m, b, SA, c.d, Sb)
    assert np.array_equal(SA, golden["cfg1_SA"]) and np.array_equal(Sb, ref["Sb"])


@pytest.mark.parametrize("kind", ["owned", "lanes"])
@pytest.mark.parametrize("keep", [False, True])
def test_host_streaming_ring_many_blocks_bitwise(kind, keep):
    """More row blocks than ring slots (64 MiB blocks of a 160 MiB A): every
    block through the two-slot ring (or in place into A_dev_keep), device
    outputs, bitwise the oracle's fold; the kept device copy equals A."""
    from oracle import clib
    from paper_2409_14309_b200._device import pinned_empty_f64
    from paper_2409_14309_b200.sketch import CountSketchPlan

    m, n, d = (1 << 20) + 4099, 20, 2048 if kind == "owned" else 5000
    rng = np.random.default_rng(7)
    A = pinned_empty_f64((m, n), fortran=True)
    A[...] = rng.standard_normal((m, n))
    b = pinned_empty_f64((m,))
    b[...] = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=8), m)
    plan = CountSketchPlan(op.rows, op.signs, d, kind=kind)
    SA = torch.full((n, d), float("nan"), dtype=torch.float64, device="cuda").t()
    Sb = torch.full((d,), float("nan"), dtype=torch.float64, device="cuda")
    ld = m + 1
    A_keep = torch.zeros((n, ld), dtype=torch.float64, device="cuda").t() if keep else None
    b_keep = torch.zeros(m, dtype=torch.float64, device="cuda") if keep else None
    plan.apply_host(A, m, n, m, b, SA, d, Sb, A_keep=A_keep, ld_keep=ld if keep else 0,
                    b_keep=b_keep)
    assert np.array_equal(SA.cpu().numpy(), clib.countsketch_apply_mt(op.rows, op.signs, d, A))
    assert np.array_equal(Sb.cpu().numpy(), clib.countsketch_apply_mt(op.rows, op.signs, d, b))
    if keep:
        assert np.array_equal(A_keep[:m].cpu().numpy(), A)
        assert np.array_equal(b_keep.cpu().numpy(), b)


def test_host_input_solve_equals_device_input_solve():
    """solve() with host carriers streams A to the device under the sketch and
    reuses the device copy for the residual: the same bits as the solve on
    device carriers."""
    c = W.config(1)
    A, b, _ = W.make_problem(c)
    spec, opts = E.SketchSpec("countsketch", 1, seed=3), E.SolverOptions(d_factor=4)
    rh = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa", spec, opts)
    rd = E.solve(E.LeastSquaresProblem(E.DenseMatrix(torch.from_numpy(A).cuda()),
                                       E.Vector(torch.from_numpy(b).cuda())), "saa", spec, opts)
    assert isinstance(rh.x.data, np.ndarray)
    assert np.array_equal(rh.x.data, rd.x.data.cpu().numpy())
    assert rh.residual_norm == rd.residual_norm


@pytest.mark.parametrize("kind", ["owned", "lanes"])
@pytest.mark.parametrize("m,n,d", [(1, 1, 1), (9, 2, 3), (8184, 3, 5), (8185, 2, 2048),
                                   (50_000, 5, 1024), (50_001, 3, 1025), (100_000, 2, 17)])
def test_countsketch_both_plans_bitwise(m, n, d, kind):
    """Both dense kernels (register-owned and lane-list) on the same
    operator: bitwise-equal to the oracle's scipy fold, ragged chunk tails,
    one-bucket and many-bucket lanes."""
    from paper_2409_14309_b200.sketch import CountSketchPlan

    rng = np.random.default_rng(m + 7 * d)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=m ^ d), m)
    plan = CountSketchPlan(op.rows, op.signs, d, kind=kind)
    lda = (m + 1) // 2 * 2  # kernels need an even leading dimension
    Ad = torch.zeros((n, lda), dtype=torch.float64, device="cuda").t()
    Ad[:m] = torch.from_numpy(A).cuda()
    bd = torch.from_numpy(b).cuda()
    SA = torch.full((n, d), float("nan"), dtype=torch.float64, device="cuda").t()
    Sb = torch.full((d,), float("nan"), dtype=torch.float64, device="cuda")
    plan.apply(Ad, m, n, lda, bd, SA, d, Sb, partitions=1)
    want = O.countsketch_apply(op.rows, op.signs, d, np.column_stack([A, b]))
    got = np.column_stack([SA.cpu().numpy(), Sb.cpu().numpy()])
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------- SRHT
@pytest.mark.parametrize("m,n,d", [(1, 1, 1), (5, 3, 2), (64, 5, 16), (1000, 7, 64),
                                   (4096, 3, 4096), (6000, 32, 256), (20_000, 9, 800),
                                   (70_000, 4, 2048)])
def test_srht_matches_oracle(m, n, d):
    rng = np.random.default_rng(m + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    op = E.build_sketch(E.SketchSpec("srht", d, seed=m), m)
    key = O.derive_seed(m, "srht", m)
    sg, rs, m_pad = O.srht_draws(key, m, d)
    assert np.array_equal(op.row_sample, rs) and np.array_equal(op.sign_diag, sg)
    want = O.srht_apply(sg, rs, m_pad, d, A)
    got = E.apply_to_matrix(op, E.DenseMatrix(A)).data
    assert rel_fro(got, want) <= 1e-13
    gv = E.apply_to_vector(op, E.Vector(A[:, 0].copy())).data
    assert rel_fro(gv, want[:, 0]) <= 1e-13


def test_srht_small_golden(golden):
    a = golden["small_A"]
    op = E.build_sketch(E.SketchSpec("srht", 16, seed=42), 64)
    assert rel_fro(E.apply_to_matrix(op, E.DenseMatrix(a)).data, golden["small_SA_srht"]) <= 1e-13


def test_srht_identity_probe_equals_materialize():
    m, d = 20, 8
    op = E.build_sketch(E.SketchSpec("srht", d, seed=21), m)
    probe = E.apply_to_matrix(op, E.DenseMatrix(np.eye(m))).data
    assert np.allclose(probe, E.materialize(op).data, rtol=1e-13, atol=1e-15)


def test_saa_srht_cfg5_reduced(golden, golden_meta):
    c, kind, A, b, ref = live_case("cfg5r", golden_meta)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                  E.SketchSpec("srht", 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n))
    assert rel_fro(res.x.data, ref["x"]) <= 1e-9
    assert abs(res.residual_norm - ref["residual"]) <= 1e-10 * ref["residual"]


def test_fwht_inplace_bitwise(golden):
    for i in range(3):
        x = golden[f"fwht_in_{i}"].copy()
        assert np.array_equal(E.fwht_inplace(x), golden[f"fwht_out_{i}"])
    x = golden["fwht_in_1024x3"].copy()
    assert np.array_equal(E.fwht_inplace(x), golden["fwht_out_1024x3"])
    big = np.random.default_rng(1).standard_normal((1 << 17, 2))
    want = O.fwht_inplace(big.copy())
    assert np.array_equal(E.fwht_inplace(big), want)


def test_fwht_rejects_bad_input():
    with pytest.raises(E.ShapeError):
        E.fwht_inplace(np.zeros(3))
    with pytest.raises(ValueError):
        E.fwht_inplace(np.zeros(4, dtype=np.float32))
    with pytest.raises(ValueError):
        E.fwht_inplace(np.asfortranarray(np.zeros((4, 2))))


# ------------------------------------------------------------------ Gaussian
def test_gaussian_entries_small_golden(golden):
    op = E.build_sketch(E.SketchSpec("gaussian", 16, seed=1), 64)
    assert np.array_equal(op.gaussian_entries, golden["gauss_16_64_1"])


@pytest.mark.parametrize("d,m", [(1, 1), (3, 5), (64, 100_003), (300, 70_000)])
def test_gaussian_entries_bitwise_numpy(d, m):
    op = E.build_sketch(E.SketchSpec("gaussian", d, seed=d + m), m)
    want = O.gaussian_draws(O.derive_seed(d + m, "gaussian", m), d, m)
    assert np.array_equal(op.gaussian_entries, want)


def test_gaussian_cfg3_operator_head_tail(golden):
    op = E.build_sketch(E.SketchSpec("gaussian", 2048, seed=3), 262_144)
    G, ldg = op.device_gaussian()
    head = G[:1, :4096].reshape(-1).cpu().numpy()
    tail = G[-1, 262_144 - 4096: 262_144].cpu().numpy()
    assert np.array_equal(head, golden["gauss_cfg3_head"])
    assert np.array_equal(tail, golden["gauss_cfg3_tail"])
    # a few full rows against the host generator's stream order
    rows = G[:3, :262_144].cpu().numpy().ravel()
    from paper_2409_14309_b200 import _native

    want = _native.rng_gaussian_host(O.derive_seed(3, "gaussian", 262_144), rows.size) / np.sqrt(2048)
    assert np.array_equal(rows, want)


@pytest.mark.parametrize("d,n,m", [(1, 1, 1), (7, 3, 5), (129, 130, 1000), (256, 64, 8192),
                                   (2048, 512, 40_000), (300, 17, 123_457)])
def test_gemm_f64_matches_numpy(d, n, m):
    rng = np.random.default_rng(d * n + m)
    G = rng.standard_normal((d, m))
    A = np.asfortranarray(rng.standard_normal((m, n)))
    ldg = (m + 31) // 32 * 32
    Gd = torch.zeros((d, ldg), dtype=torch.float64, device="cuda")
    Gd[:, :m] = torch.from_numpy(G).cuda()
    Ad = torch.from_numpy(A).cuda()
    lda = m if n == 1 else int(Ad.stride(1))
    if lda % 2:
        Ad = torch.zeros((n, m + 1), dtype=torch.float64, device="cuda").t()[:m]
        Ad.copy_(torch.from_numpy(A).cuda())
        lda = m + 1
    C = torch.zeros((n, d), dtype=torch.float64, device="cuda").t()
    _native.call("skl_gemm_f64", Gd.data_ptr(), ldg, Ad.data_ptr(), lda, C.data_ptr(), d, d, n, m,
                 0, torch.cuda.current_stream().cuda_stream)
    want = G @ A
    assert rel_fro(C.cpu().numpy(), want) <= 1e-14


def test_gaussian_apply_small_golden(golden):
    a = golden["small_A"]
    op = E.build_sketch(E.SketchSpec("gaussian", 16, seed=42), 64)
    assert rel_fro(E.apply_to_matrix(op, E.DenseMatrix(a)).data, golden["small_SA_gaussian"]) <= 1e-14
    assert rel_fro(E.apply_to_vector(op, E.Vector(a[:, 0].copy())).data,
                   golden["small_Sb_gaussian"]) <= 1e-14


def test_saa_gaussian_cfg3_reduced(golden, golden_meta):
    c, kind, A, b, ref = live_case("cfg3r", golden_meta)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                  E.SketchSpec("gaussian", 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n))
    assert rel_fro(res.x.data, ref["x"]) <= 1e-9
    assert abs(res.residual_norm - ref["residual"]) <= 1e-10 * ref["residual"]
    assert rel_fro(res.x.data, golden["cfg3r_x"]) <= 1e-9


# ------------------------------------------------------------ reduced solve
@pytest.mark.parametrize("d,n", [(64, 31), (64, 33), (300, 100), (2048, 256), (1500, 400),
                                 (2048, 513), (8192, 1024), (12_000, 64), (20_000, 40)])
def test_qr_solve_matches_lapack(d, n):
    rng = np.random.default_rng(d + n)
    M = rng.standard_normal((d, n)) @ np.diag(np.logspace(0, -6, n))
    y = rng.standard_normal(d)
    from paper_2409_14309_b200.linalg import qr_solve_device

    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    yd = torch.from_numpy(y).cuda()
    x, R, Q = qr_solve_device(Md, d, yd, d, n, want_q=True, want_r=True)
    R, Q, x = R.cpu().numpy(), Q.cpu().numpy(), x.cpu().numpy()
    q_ref, r_ref = O.economy_qr(M)
    assert np.all(np.diagonal(R) >= 0) and np.array_equal(np.tril(R, -1), np.zeros((n, n)))
    assert rel_fro(R, r_ref) <= 1e-12
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-12
    assert rel_fro(Q @ R, M) <= 1e-13
    x_ref = np.linalg.lstsq(M, y, rcond=None)[0]
    assert rel_fro(x, x_ref) <= 1e-8


@pytest.mark.parametrize("m,n,d,density,dense_rows", [
    (1, 1, 1, 1.0, 0), (50, 7, 3, 0.5, 0), (5000, 40, 64, 0.02, 3), (20_000, 1024, 256, 1e-3, 0),
    (30_000, 3000, 8, 2e-3, 1), (100_000, 64, 2048, 0.0, 0), (70_000, 300, 1024, 0.01, 2)])
def test_countsketch_csr_kernel_bitwise(m, n, d, density, dense_rows):
    """CSR operand: bitwise-equal to scipy's (S @ A).toarray() (csr_matmat
    order) -- empty matrix/rows, fully dense rows (more nonzeros than one
    staging pass), buckets with many rows, several column tiles."""
    rng = np.random.default_rng(m + n + d)
    A = scipy.sparse.random(m, n, density=density, format="csr", random_state=rng,
                            data_rvs=rng.standard_normal)
    if dense_rows:
        A = A.tolil()
        for r in rng.choice(m, size=dense_rows, replace=False):
            A[r, :] = rng.standard_normal(n)
        A = A.tocsr()
    A.sort_indices()
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=m ^ n), m)
    got = E.apply_to_matrix(op, E.SparseMatrix.from_scipy(A)).data
    want = O.countsketch_apply(op.rows.astype(np.int64), op.signs.astype(np.float64), d, A)
    assert np.array_equal(np.asarray(got), want)


@pytest.mark.parametrize("kind,m,n,d,world", [
    ("countsketch", 50_000, 7, 512, 3), ("srht", 40_000, 5, 256, 2), ("srht", 1 << 16, 3, 512, 4),
    ("gaussian", 30_000, 6, 128, 3)])
def test_row_shards_sum_to_full_apply(kind, m, n, d, world):
    """Multi-GPU partials computed one shard at a time on one GPU (no
    collectives): the sum over shards equals the single-device S[A|b]
    (CountSketch/SRHT/Gaussian shard plans: global hashes, SRHT block offsets,
    Gaussian column blocks)."""
    from paper_2409_14309_b200.distributed import ShardPlan, local_partial_device, shard_rows

    rng = np.random.default_rng(m + d)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec(kind, d, seed=11), m)
    total = None
    for r in range(world):
        r0, r1 = shard_rows(m, world, r)
        if r1 <= r0:
            continue
        Ad = torch.from_numpy(np.asfortranarray(A[r0:r1])).cuda()
        bd = torch.from_numpy(b[r0:r1].copy()).cuda()
        part = local_partial_device(ShardPlan(op, r0, r1), Ad, r1 - r0, bd).cpu().numpy()
        total = part if total is None else total + part
    full = np.column_stack([E.apply_to_matrix(op, E.DenseMatrix(A)).data,
                            E.apply_to_vector(op, E.Vector(b)).data])
    assert rel_fro(total, full) <= 1e-13


SAP_GPU_CASES = {
    "sap_cfg1": (W.config(1), "countsketch", True),
    "sap_cfg2r": (W.config(2, m=1 << 14), "countsketch", True),
    "sap_cfg3r": (W.config(3, m=8192, n=64, d=256), "gaussian", True),
    "sap_cfg4r": (W.config(4, m=1 << 16, n=256, d=2048), "countsketch", True),
    "sap_cfg5r": (W.config(5, m=6000, n=32, d=256), "srht", False),
}


@pytest.mark.parametrize("name", list(SAP_GPU_CASES))
def test_sap_matches_oracle(golden_meta, name):
    """solve(problem, "sap", ...): sketch -> device QR (R) -> warm start ->
    device LSQR preconditioned by R (solvers.py:323-361, 110-255) against the
    oracle on the same inputs: same iteration count and stopping rule, x and
    ||Ax - b|| to 1e-9 / 1e-10."""
    c, kind, warm = SAP_GPU_CASES[name]
    A, b, _ = W.make_problem(c)
    want = O.sap_solve(A, b, kind, W.SEED, c.d / c.n, warm_start=warm)
    Ac = E.SparseMatrix.from_scipy(A) if scipy.sparse.issparse(A) else E.DenseMatrix(A)
    res = E.solve(E.LeastSquaresProblem(Ac, E.Vector(b)), "sap",
                  E.SketchSpec(kind, 1, seed=W.SEED),
                  E.SolverOptions(d_factor=c.d / c.n, warm_start=warm))
    assert res.method == "sap" and res.sketch == kind and res.d == c.d
    assert res.termination == want["termination"]
    assert abs(res.iterations - want["iterations"]) <= 1, (res.iterations, want["iterations"])
    # cfg2 is kappa = 1e8: any backward-stable solve moves x by ~kappa*eps ~ 1e-8
    # (SURVEY.md §7 H2); the residual still agrees to 1e-10
    x_tol = 5e-8 if name == "sap_cfg2r" else 1e-9
    assert rel_fro(res.x.data, want["x"]) <= x_tol
    assert abs(res.residual_norm - want["residual"]) <= 1e-10 * want["residual"]
    assert golden_meta[f"{name}_iterations"] == want["iterations"]


def test_plain_lsqr_matches_oracle():
    c = W.config(1, m=3000, n=40)
    A, b, _ = W.make_problem(c)
    want = O.lsqr(np.asfortranarray(A), b)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "lsqr")
    assert res.method == "lsqr" and res.termination == want["termination"]
    assert abs(res.iterations - want["iterations"]) <= 1
    assert rel_fro(res.x.data, want["x"]) <= 1e-9
    assert abs(res.residual_norm - want["residual"]) <= 1e-10 * want["residual"]


def test_sap_device_resident_and_sparse_lsqr():
    c = W.config(1, m=4000, n=30)
    A, b, _ = W.make_problem(c)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(Ad), E.Vector(torch.from_numpy(b).cuda())),
                  "sap", E.SketchSpec("countsketch", 1, seed=3))
    assert res.x.data.is_cuda
    want = O.sap_solve(A, b, "countsketch", 3, 4.0)
    assert rel_fro(res.x.data.cpu().numpy(), want["x"]) <= 1e-9
    # plain LSQR on a CSR operand (CSC transposed product on the device)
    rng = np.random.default_rng(3)
    S = scipy.sparse.random(5000, 40, density=0.05, format="csr", random_state=rng,
                            data_rvs=rng.standard_normal)
    bs = rng.standard_normal(5000)
    want = O.lsqr(S, bs)
    res = E.solve(E.LeastSquaresProblem(E.SparseMatrix.from_scipy(S), E.Vector(bs)), "lsqr")
    assert res.termination == want["termination"]
    assert abs(res.iterations - want["iterations"]) <= 1
    assert rel_fro(res.x.data, want["x"]) <= 1e-9


def test_lsqr_edge_cases():
    """Zero right-hand side (x = 0, no iterations) and the max_iter stop,
    against the oracle's LSQR (solvers.py:176-189, 232-233)."""
    c = W.config(1, m=2000, n=25)
    A, b, _ = W.make_problem(c)
    prob0 = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(np.zeros(2000)))
    res = E.solve(prob0, "lsqr")
    assert res.iterations == 0 and res.termination == "atol_btol"
    assert np.array_equal(res.x.data, np.zeros(25))
    want = O.lsqr(np.asfortranarray(A), b, max_iter=3)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "lsqr",
                  opts=E.SolverOptions(max_iter=3))
    assert res.iterations == 3 and res.termination == "max_iter" == want["termination"]
    assert rel_fro(res.x.data, want["x"]) <= 1e-12
    # sap without warm start on a device-resident problem, tight max_iter
    want = O.sap_solve(A, b, "countsketch", 2, 4.0, warm_start=False, max_iter=2)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "sap",
                  E.SketchSpec("countsketch", 1, seed=2),
                  E.SolverOptions(warm_start=False, max_iter=2))
    assert res.iterations == 2 and res.termination == "max_iter"
    assert rel_fro(res.x.data, want["x"]) <= 1e-10


@pytest.mark.parametrize("m,d", [(1, 1), (7, 2), (20_000, 800), (1 << 20, 2048), (123_457, 3),
                                 (4000, 3 << 29)])
def test_device_countsketch_draws_match_host(m, d):
    """skl_rng_countsketch_device == the host walk (== numpy), including the
    forced-rejection stream (d = 3*2^29: a quarter of the draws rejected)
    that takes the host path."""
    key = O.derive_seed(77, "countsketch", m)
    rows_d = torch.empty(m, dtype=torch.int32, device="cuda")
    signs_d = torch.empty(m, dtype=torch.int8, device="cuda")
    _native.call("skl_rng_countsketch_device", key, m, d, rows_d.data_ptr(), signs_d.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    rows, signs = _native.rng_countsketch(key, m, d)
    assert np.array_equal(rows_d.cpu().numpy(), rows)
    assert np.array_equal(signs_d.cpu().numpy(), signs)


@pytest.mark.parametrize("m,d", [(1, 1), (100, 4), (8185, 5), (20_000, 800), (65_537, 2048),
                                 (1 << 20, 2048), (30_001, 1025)])
def test_device_owned_plan_matches_host(m, d):
    """The device plan builder emits the host planner's words exactly
    (bitonic bucket sort + the same greedy bank-balancing merge), including
    the chunk shrink for tiny d."""
    from paper_2409_14309_b200.sketch import CountSketchPlan

    E.clear_operator_cache()
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=m + d), m)
    rows, signs = op.rows, op.signs  # host copies of the device draws
    key = O.derive_seed(m + d, "countsketch", m)
    want_rows, want_signs = O.countsketch_draws(key, m, d)
    assert np.array_equal(rows, want_rows) and np.array_equal(signs, want_signs)
    dev = op.device_plan()
    host = CountSketchPlan(rows, signs, d)
    assert (dev.chunk, dev.warps, dev.max_block) == (host.chunk, host.warps, host.max_block)
    assert np.array_equal(dev.off.cpu().numpy(), host.off.cpu().numpy())
    n = host.lanes.numel()
    assert np.array_equal(dev.lanes[:n].cpu().numpy(), host.lanes.cpu().numpy())


@pytest.mark.parametrize("m,n,d,s", [(1, 1, 1, 1), (60, 3, 32, 5), (40, 2, 9, 8), (3000, 7, 64, 8),
                                     (20_000, 200, 800, 8), (65_537, 5, 2048, 8),
                                     (10_000, 4, 512, 1), (5000, 3, 100, 100)])
def test_sparsesign_dense_apply_bitwise(m, n, d, s):
    """Sparse sign embedding S A, S b on the device (register-owned plan with
    s entries per row, one rounded product per entry) against scipy's
    csr_matvecs fold: bitwise."""
    rng = np.random.default_rng(m + s)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec("sparsesign", d, seed=m + d, sparsity=s), m)
    smap = op.sparse_map
    assert np.array_equal(E.apply_to_matrix(op, E.DenseMatrix(A)).data, smap @ A)
    assert np.array_equal(E.apply_to_vector(op, E.Vector(b)).data, smap @ b)


@pytest.mark.parametrize("m,n,d,s", [(3000, 40, 64, 8), (20_000, 300, 4096, 8), (500, 9, 9, 8)])
def test_sparsesign_csr_apply_bitwise(m, n, d, s):
    rng = np.random.default_rng(m)
    A = scipy.sparse.random(m, n, density=0.05, format="csr", random_state=rng,
                            data_rvs=rng.standard_normal)
    A.sort_indices()
    op = E.build_sketch(E.SketchSpec("sparsesign", d, seed=3, sparsity=s), m)
    got = E.apply_to_matrix(op, E.SparseMatrix.from_scipy(A)).data
    assert np.array_equal(np.asarray(got), (op.sparse_map @ A).toarray())


def test_sparsesign_saa_and_limits(golden, golden_meta):
    c = W.config(1)
    A, b, _ = W.make_problem(c)
    want = O.saa_solve(A, b, "sparsesign", W.SEED, c.d / c.n)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                  E.SketchSpec("sparsesign", 1, seed=W.SEED), E.SolverOptions(d_factor=c.d / c.n))
    assert res.sketch == "sparsesign" and res.d == c.d
    assert rel_fro(res.x.data, want["x"]) <= 1e-9
    assert abs(res.residual_norm - want["residual"]) <= 1e-10 * want["residual"]
    assert rel_fro(want["x"], golden["ss_cfg1_x"]) <= 1e-12
    # dense operands with d > 2048: shared-memory lane-list plan, s entries per row
    rng = np.random.default_rng(4)
    A2 = rng.standard_normal((10_000, 3))
    op = E.build_sketch(E.SketchSpec("sparsesign", 4096, seed=1), 10_000)
    assert np.array_equal(E.apply_to_matrix(op, E.DenseMatrix(A2)).data, op.sparse_map @ A2)


@pytest.mark.parametrize("m,n,d,s", [(30_000, 6, 3000, 8), (20_001, 3, 8192, 4), (5000, 2, 2049, 1),
                                     (9000, 5, 4500, 16)])
def test_sparsesign_dense_large_d_bitwise(m, n, d, s):
    """Sparse sign embeddings with d > 2048 on dense operands (lane-list plan
    with s entries per source row, SCALED kernel): bitwise to scipy."""
    rng = np.random.default_rng(m + d)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec("sparsesign", d, seed=d, sparsity=s), m)
    assert np.array_equal(E.apply_to_matrix(op, E.DenseMatrix(A)).data, op.sparse_map @ A)
    assert np.array_equal(E.apply_to_vector(op, E.Vector(b)).data, op.sparse_map @ b)


def test_sparsesign_saa_large_n():
    """method "saa" with a sparse sign embedding at n = 600 (d = 2400 > 2048)."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((20_000, 600))
    b = A @ rng.standard_normal(600) + 1e-3 * rng.standard_normal(20_000)
    want = O.saa_solve(A, b, "sparsesign", 5, 4.0)
    res = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                  E.SketchSpec("sparsesign", 1, seed=5), E.SolverOptions(d_factor=4.0))
    assert res.d == 2400 == want["d"]
    assert rel_fro(res.x.data, want["x"]) <= 1e-9


def test_concurrent_solves_from_threads():
    """The C-ABI is reentrant (SURVEY.md §8b threading): four host threads
    solving different problems at once, each on its own CUDA stream, get the
    same answers as serial solves."""
    import threading

    cases = []
    for t in range(4):
        c = W.config(1, m=6000 + 1000 * t, n=20 + t)
        A, b, _ = W.make_problem(c, seed=100 + t)
        cases.append((A, b, "countsketch" if t % 2 == 0 else "srht"))
    serial = [E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                      E.SketchSpec(kind, 1, seed=5)).x.data for A, b, kind in cases]
    out = [None] * 4
    errs = []

    def work(t):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                A, b, kind = cases[t]
                r = E.solve(E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b)), "saa",
                            E.SketchSpec(kind, 1, seed=5))
                torch.cuda.current_stream().synchronize()
                out[t] = r.x.data
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errs, errs
    for t in range(4):
        assert np.array_equal(out[t], serial[t])


def test_lsqr_with_preconditioner_and_callback():
    """lsqr(A, b, opts, precond_R, callback) as solvers.py:110-255: the
    preconditioned iteration matches the oracle, the callback sees every
    iteration with a nonincreasing residual estimate."""
    rng = np.random.default_rng(11)
    A = rng.standard_normal((3000, 24)) @ np.diag(np.logspace(0, -4, 24))
    b = rng.standard_normal(3000)
    R = np.linalg.qr(A[rng.choice(3000, 200, replace=False)], mode="r")
    R = np.triu(R)
    want = O.lsqr(A, b, precond_R=R)
    seen = []
    res = E.lsqr(E.DenseMatrix(A), E.Vector(b), precond_R=E.DenseMatrix(R),
                 callback=lambda itn, x, rn: seen.append((itn, x.shape, rn)))
    assert res.method == "lsqr" and res.iterations == want["iterations"]
    assert rel_fro(res.x.data, want["x"]) < 1e-9
    assert [s[0] for s in seen] == list(range(1, res.iterations + 1))
    assert all(s[1] == (24,) for s in seen)
    rn = [s[2] for s in seen]
    assert all(rn[i + 1] <= rn[i] * (1 + 1e-12) for i in range(len(rn) - 1))


@pytest.mark.parametrize("m,n,d", [(40_000, 3, 10_000), (20_000, 2, 16_385)])
def test_srht_more_rows_than_one_launch(m, n, d):
    """SRHT with d > 8192 sampled rows: one pass over A per 8192-row slice of
    row_sample, all normalised by the whole 1/sqrt(d)."""
    rng = np.random.default_rng(d)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    op = E.build_sketch(E.SketchSpec("srht", d, seed=2), m)
    got = E.apply_to_matrix(op, E.DenseMatrix(A)).data
    want, _ = O.sketch_apply("srht", O.operator_key(2, "srht", m), d, A)
    assert rel_fro(got, want) <= 1e-13


def test_qr_solve_wide_system():
    """n above the 48 KB default shared-memory window of the back-solve
    (n = 6400: y takes 51 KB)."""
    from paper_2409_14309_b200.linalg import qr_solve_device

    rng = np.random.default_rng(64)
    d, n = 6600, 6400
    M = rng.standard_normal((d, n)) + 4 * np.eye(d, n)
    y = rng.standard_normal(d)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    x, _, _ = qr_solve_device(Md, d, torch.from_numpy(y).cuda(), d, n)
    want = np.linalg.lstsq(M, y, rcond=None)[0]
    assert rel_fro(x.cpu().numpy(), want) <= 1e-10


@pytest.mark.parametrize("m,n,d", [(1 << 16, 5, 256), (100_000, 3, 64), (1 << 20, 1, 2048)])
def test_srht_ab_single_pass(m, n, d):
    """S [A | b] in one SRHT pass (b as the last column, the SAA solve's
    path) against the oracle's separate applies; a single long column (the
    vector apply, split over enough CTAs to fill the GPU) too."""
    from paper_2409_14309_b200.sketch import _srht_device_ab

    rng = np.random.default_rng(m + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec("srht", d, seed=m ^ d), m)
    SA, Sb = _srht_device_ab(op, torch.from_numpy(A).cuda(), m, n, torch.from_numpy(b).cuda())
    ref_A, ref_b = O.sketch_apply("srht", O.derive_seed(m ^ d, "srht", m), d, A, b)
    assert rel_fro(SA.cpu().numpy(), ref_A) <= 1e-13
    assert rel_fro(Sb.cpu().numpy(), ref_b) <= 1e-13
    v = E.apply_to_vector(op, E.Vector(torch.from_numpy(b).cuda())).data.cpu().numpy()
    assert rel_fro(v, ref_b) <= 1e-13


@pytest.mark.parametrize("kind", ["countsketch", "srht", "gaussian"])
def test_apply_captures_in_cuda_graph(kind):
    """A warmed-up apply captures in a CUDA graph (the cached operator's
    artifacts are not waited on inside the capture) and replays exactly."""
    m, n, d = 50_000, 6, 256
    A = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    op = E.build_sketch(E.SketchSpec(kind, d, seed=3), m)
    from paper_2409_14309_b200.sketch import _apply_dense_tensor

    want = _apply_dense_tensor(op, A, m, n, lda=m).clone()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = _apply_dense_tensor(op, A, m, n, lda=m)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)
