"""Device problem generation, the direct method, the linalg helpers, the
CLI on the GPU, against fixtures the
reference produced (tests/golden/golden.npz, tests/golden/io/)."""

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_fro

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native, cli  # noqa: E402
from paper_2409_14309_b200.probgen import _NormalStream  # noqa: E402

IO = Path(__file__).resolve().parent / "golden" / "io"


def test_normals_resume_at_the_stream_word():
    key = 0x9E3779B97F4A7C15
    n1, n2, n3 = 1000, 4097, 77
    want = _native.rng_gaussian_host(key, n1 + n2 + n3)
    s = _NormalStream(key)
    a = s.draw(10, 100).cpu().numpy().ravel()
    b = s.draw(17, 241).cpu().numpy().ravel()
    c = s.draw(1, n3).cpu().numpy().ravel()
    got = np.concatenate([a, b, c])
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("name", ["pg_tall", "pg_square", "pg_col", "pg_default"])
def test_generate_problem_matches_reference(golden, golden_meta, name):
    m, n, kappa, beta, seed = golden_meta[f"{name}_spec"]
    prob = E.generate_problem(E.ProblemSpec(m=m, n=n, kappa=kappa, beta=beta, seed=seed))
    assert prob.A.on_device and prob.b.on_device and prob.beta == beta
    A = prob.A.to_numpy()
    # same normals bit for bit; QR/GEMM on cuSOLVER/cuBLAS vs OpenBLAS -> rounding only
    assert prob.x_star.to_numpy().tobytes() == golden[f"{name}_xstar"].tobytes()
    assert rel_fro(A, golden[f"{name}_A"]) < 1e-13
    assert rel_fro(prob.b.to_numpy(), golden[f"{name}_b"]) < 1e-13
    # the construction's promises: x_star is the minimiser, beta the optimal residual
    r = A @ prob.x_star.to_numpy() - prob.b.to_numpy()
    assert abs(np.linalg.norm(r) - beta) <= 1e-12 * max(1.0, np.linalg.norm(prob.b.to_numpy()))
    s = np.linalg.svd(A, compute_uv=False)
    want_kappa = kappa if n > 1 else 1.0  # n == 1: sigma = [1] (probgen.py:56-57)
    assert abs(s[0] / s[-1] - want_kappa) / want_kappa < 1e-3


def test_generate_problem_is_deterministic():
    spec = E.ProblemSpec(m=257, n=16, kappa=1e8, beta=1e-6, seed=5)
    p1, p2 = E.generate_problem(spec), E.generate_problem(spec)
    assert p1.A.to_numpy().tobytes() == p2.A.to_numpy().tobytes()
    assert p1.b.to_numpy().tobytes() == p2.b.to_numpy().tobytes()


def test_direct_method_matches_reference(golden, golden_meta):
    from paper_2409_14309_b200 import workloads as W

    A, b, _ = W.make_problem(W.config(1, m=3000, n=40))
    res = E.solve(E.LeastSquaresProblem(A=E.DenseMatrix(A), b=E.Vector(b)), "direct")
    assert res.method == "direct" and res.termination == "direct" and res.sketch is None
    assert rel_fro(res.x.data, golden["direct_small_x"]) < 1e-12
    assert abs(res.residual_norm - golden_meta["direct_small_residual"]) <= \
        1e-10 * golden_meta["direct_small_residual"]


def test_direct_method_sparse_and_device():
    rng = np.random.default_rng(3)
    import scipy.sparse

    S = scipy.sparse.random(400, 12, density=0.2, random_state=4, format="csr")
    b = rng.standard_normal(400)
    want = np.linalg.lstsq(S.toarray(), b, rcond=None)[0]
    res = E.solve(E.LeastSquaresProblem(A=E.SparseMatrix.from_scipy(S), b=E.Vector(b)), "direct")
    assert rel_fro(res.x.data, want) < 1e-12
    Ad = torch.from_numpy(np.asfortranarray(S.toarray())).cuda().t().contiguous().t()
    res2 = E.solve(E.LeastSquaresProblem(A=E.DenseMatrix(Ad), b=E.Vector(torch.from_numpy(b).cuda())),
                   "direct")
    assert rel_fro(res2.x.data.cpu().numpy(), want) < 1e-12
    x = E.normal_equations_oracle(E.DenseMatrix(S.toarray()), E.Vector(b))
    assert rel_fro(x.data, want) < 1e-12


def test_default_method_is_lsqr_like_the_reference():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((500, 10))
    b = rng.standard_normal(500)
    res = E.solve(E.LeastSquaresProblem(A=E.DenseMatrix(A), b=E.Vector(b)))
    assert res.method == "lsqr" and res.iterations > 0


def test_products_and_triangular_solves():
    rng = np.random.default_rng(7)
    import scipy.sparse

    A = rng.standard_normal((1001, 37))
    x = rng.standard_normal(37)
    y = rng.standard_normal(1001)
    assert rel_fro(E.matvec(E.DenseMatrix(A), E.Vector(x)).data, A @ x) < 1e-14
    assert rel_fro(E.matvec_transpose(E.DenseMatrix(A), E.Vector(y)).data, A.T @ y) < 1e-14
    S = scipy.sparse.random(1001, 37, density=0.05, random_state=1, format="csr")
    Ss = E.SparseMatrix.from_scipy(S)
    assert rel_fro(E.matvec(Ss, E.Vector(x)).data, S @ x) < 1e-14
    assert rel_fro(E.matvec_transpose(Ss, E.Vector(y)).data, S.T @ y) < 1e-14
    Ad = torch.from_numpy(A).cuda().t().contiguous().t()
    got = E.matvec(E.DenseMatrix(Ad), E.Vector(torch.from_numpy(x).cuda()))
    assert got.on_device and rel_fro(got.data.cpu().numpy(), A @ x) < 1e-14
    with pytest.raises(E.ShapeError, match="matvec: A is 1001x37 but x has length 36"):
        E.matvec(E.DenseMatrix(A), E.Vector(x[:36]))
    R = np.triu(rng.standard_normal((37, 37))) + 5 * np.eye(37)
    import scipy.linalg

    for tr in (False, True):
        z = E.solve_triangular(E.DenseMatrix(R), E.Vector(x), transposed=tr).data
        want = scipy.linalg.solve_triangular(R, x, trans="T" if tr else "N")
        assert rel_fro(z, want) < 1e-13
    R0 = R.copy()
    R0[4, 4] = 0.0
    with pytest.raises(E.SingularFactorError, match="zero diagonal entry at index 4"):
        E.solve_triangular(E.DenseMatrix(R0), E.Vector(x))
    k = E.spectral_condition_number(E.DenseMatrix(A))
    s = np.linalg.svd(A, compute_uv=False)
    assert abs(k - s[0] / s[-1]) / k < 1e-10


def test_cli_gen_then_solve(tmp_path, capsys):
    out = tmp_path / "p"
    assert cli.main(["gen", "--m", "600", "--n", "12", "--cond", "1e6", "--beta", "1e-8",
                     "--seed", "9", "--out", str(out)]) == 0
    prob, meta = E.read_problem_dir(str(out))
    assert meta["m"] == "600" and meta["seed"] == "9"
    for method in ("saa", "sap", "lsqr", "direct"):
        xf = tmp_path / f"x_{method}.mtx"
        rc = cli.main(["solve", "--A", str(out / "A.mtx"), "--b", str(out / "b.mtx"),
                       "--method", method, "--json", "--out", str(xf), "--seed", "2"])
        assert rc == 0
        summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        assert summary["method"] == method
        x = E.read_vector(str(xf)).data
        fe = np.linalg.norm(x - prob.x_star.data) / np.linalg.norm(prob.x_star.data)
        assert fe < (1e-2 if method == "saa" else 1e-6), (method, fe)
    # key=value output
    assert cli.main(["solve", "--A", str(out / "A.mtx"), "--b", str(out / "b.mtx"),
                     "--method", "saa"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "method=saa" and any(ln.startswith("d=48") for ln in lines)


def test_cli_numerical_failure_exit_code(tmp_path, capsys):
    A = np.ones((20, 3))
    E.write_matrix(str(tmp_path / "A.mtx"), E.DenseMatrix(A))
    E.write_vector(str(tmp_path / "b.mtx"), E.Vector(np.ones(20)))
    rc = cli.main(["solve", "--A", str(tmp_path / "A.mtx"), "--b", str(tmp_path / "b.mtx"),
                   "--method", "saa"])
    assert rc == cli.EXIT_NUMERICAL
    assert "numerical failure" in capsys.readouterr().err


def test_readme_example_runs():
    """The README's Python snippet, executed as written."""
    text = (Path(__file__).resolve().parents[1] / "README.md").read_text()
    code = text.split("```python\n", 1)[1].split("```", 1)[0]
    ns: dict = {}
    exec(compile(code, "README.md", "exec"), ns)
    assert ns["res"].d == 2048 and ns["res"].method == "saa"
    assert ns["SA"].rows == 800 and ns["SA"].cols == 200
