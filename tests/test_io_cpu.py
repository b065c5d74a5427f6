"""Matrix Market, problem directories and the CLI front
end on the host: byte-for-byte against files the
reference wrote (tests/golden/io/, made by tests/golden/make_golden.py), the
reference's error behaviour, and the CLI's exit codes -- including that a
solve without a GPU fails loudly instead of falling back to the CPU."""

import json
from pathlib import Path

import numpy as np
import pytest

import torch

import paper_2409_14309_b200 as E
from paper_2409_14309_b200 import cli

IO = Path(__file__).resolve().parent / "golden" / "io"


def _bytes(p):
    return Path(p).read_bytes()


DENSE = np.array([[0.1, -2.5e-7], [1e16, 5e-324], [-0.0, 123456789.0], [1.0 / 3.0, -7.0]])


def test_write_dense_sparse_vector_match_reference_bytes(tmp_path):
    E.write_matrix(str(tmp_path / "dense.mtx"), E.DenseMatrix(DENSE))
    sp = E.SparseMatrix(4, 3, np.array([0, 1, 1, 3, 4]), np.array([1, 0, 2, 1]),
                        np.array([1.5, -2.0, 1e-300, 3.25]))
    E.write_matrix(str(tmp_path / "sparse.mtx"), sp)
    E.write_vector(str(tmp_path / "vector.mtx"), E.Vector(np.array([2.0, -0.5, 1e-9])))
    for name in ("dense.mtx", "sparse.mtx", "vector.mtx"):
        assert _bytes(tmp_path / name) == _bytes(IO / name), name


def test_read_round_trip_is_bitwise():
    A = E.read_matrix(str(IO / "dense.mtx"))
    assert isinstance(A, E.DenseMatrix)
    assert A.data.tobytes() == np.asfortranarray(DENSE).tobytes()
    S = E.read_matrix(str(IO / "sparse.mtx"))
    assert isinstance(S, E.SparseMatrix)
    np.testing.assert_array_equal(S.indptr, [0, 1, 1, 3, 4])
    np.testing.assert_array_equal(S.indices, [1, 0, 2, 1])
    assert S.values.tobytes() == np.array([1.5, -2.0, 1e-300, 3.25]).tobytes()
    v = E.read_vector(str(IO / "vector.mtx"))
    assert v.data.tobytes() == np.array([2.0, -0.5, 1e-9]).tobytes()
    # a sparse single column reads as a vector too
    assert E.read_vector(str(IO / "sparse.mtx").replace("sparse", "vector")).len == 3


def test_coordinate_canonicalisation_matches_reference(golden):
    S = E.read_matrix(str(IO / "dups.mtx"))
    np.testing.assert_array_equal(S.indptr, golden["io_dups_indptr"])
    np.testing.assert_array_equal(S.indices, golden["io_dups_indices"])
    np.testing.assert_array_equal(S.values, golden["io_dups_values"])


@pytest.mark.parametrize("text,msg", [
    ("", "missing %%MatrixMarket header"),
    ("%%MatrixMarket matrix array real\n1 1\n1\n", "malformed header"),
    ("%%MatrixMarket vector array real general\n1 1\n1\n", "malformed header"),
    ("%%MatrixMarket matrix csr real general\n1 1\n1\n", "unsupported format"),
    ("%%MatrixMarket matrix array complex general\n1 1\n1\n", "unsupported field"),
    ("%%MatrixMarket matrix array real symmetric\n1 1\n1\n", "unsupported symmetry"),
    ("%%MatrixMarket matrix array real general\n", "missing size line"),
    ("%%MatrixMarket matrix array real general\n2 x\n1\n", "bad array size line"),
    ("%%MatrixMarket matrix array real general\n2 1\n1\n", "expected 2 entries, found 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", "bad coordinate size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n", "bad coordinate entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "expected 2 entries"),
])
def test_malformed_files_raise_value_error(tmp_path, text, msg):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        E.read_matrix(str(p))


def test_read_vector_rejects_matrices():
    with pytest.raises(E.ShapeError, match="expected a single-column matrix, got 4x2"):
        E.read_vector(str(IO / "dense.mtx"))


def test_problem_dir_round_trip_matches_reference(tmp_path):
    prob, meta = E.read_problem_dir(str(IO / "problem"))
    assert meta == {"m": "30", "n": "4", "kappa": "10000.0", "beta": "1e-06", "seed": "11"}
    assert prob.beta == 1e-6 and prob.A.rows == 30 and prob.A.cols == 4
    spec = E.ProblemSpec(m=30, n=4, kappa=1e4, beta=1e-6, seed=11)
    E.write_problem_dir(spec, prob, str(tmp_path / "p"))
    for name in ("A.mtx", "b.mtx", "xstar.mtx", "meta.txt"):
        assert _bytes(tmp_path / "p" / name) == _bytes(IO / "problem" / name), name


def test_problem_spec_validation():
    with pytest.raises(E.SpecError, match="need m >= n >= 1"):
        E.ProblemSpec(m=3, n=5)
    with pytest.raises(E.SpecError, match="kappa must be >= 1"):
        E.ProblemSpec(m=5, n=3, kappa=0.5)
    with pytest.raises(E.SpecError, match="beta must be >= 0"):
        E.ProblemSpec(m=5, n=3, beta=float("nan"))
    # checked before any device work (probgen.py:46-50)
    with pytest.raises(E.InfeasibleResidualError, match="m >= n\\+1"):
        E.generate_problem(E.ProblemSpec(m=4, n=4, beta=1e-3))


# ---------------------------------------------------------------- CLI exit codes
def test_cli_usage_errors(capsys, monkeypatch):
    assert cli.main(["gen", "--m", "3", "--n", "5", "--out", "/tmp/x"]) == cli.EXIT_USAGE
    assert "need m >= n >= 1" in capsys.readouterr().err
    monkeypatch.setenv("SKETCHLS_SEED", "abc")
    assert cli.main(["gen", "--m", "8", "--n", "2", "--out", "/tmp/x"]) == cli.EXIT_USAGE
    assert "SKETCHLS_SEED must be an integer" in capsys.readouterr().err
    with pytest.raises(SystemExit) as ex:
        cli.main(["solve", "--A", "a.mtx"])
    assert ex.value.code == 2


def test_cli_io_error(tmp_path, capsys):
    rc = cli.main(["solve", "--A", str(tmp_path / "missing.mtx"), "--b", str(IO / "vector.mtx")])
    assert rc == cli.EXIT_IO
    assert "missing.mtx" in capsys.readouterr().err


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_cli_solve_without_gpu_fails_loudly(capsys):
    prob = IO / "problem"
    rc = cli.main(["solve", "--A", str(prob / "A.mtx"), "--b", str(prob / "b.mtx"),
                   "--method", "saa", "--json"])
    assert rc == cli.EXIT_USAGE
    assert "CUDA" in capsys.readouterr().err


def test_module_entry_point_help():
    import subprocess
    import sys

    out = subprocess.run([sys.executable, "-m", "paper_2409_14309_b200", "--help"],
                         capture_output=True, text=True, cwd=str(Path(__file__).resolve().parents[1]))
    assert out.returncode == 0 and "{gen,solve}" in out.stdout
    json.dumps({})  # keep the json import exercised for the GPU twin of this file
