"""API-level argument checks that run before any device work (no GPU)."""

import numpy as np
import pytest

import paper_2409_14309_b200 as E


def _prob(m=40, n=5):
    rng = np.random.default_rng(0)
    return E.DenseMatrix(rng.standard_normal((m, n))), E.Vector(rng.standard_normal(m))


def test_lsqr_preconditioner_validation():
    A, b = _prob()
    with pytest.raises(E.ShapeError, match="preconditioner must be 5x5, got 4x4"):
        E.lsqr(A, b, precond_R=E.DenseMatrix(np.eye(4)))
    low = np.eye(5)
    low[3, 1] = 0.5
    with pytest.raises(E.ShapeError, match="preconditioner must be upper triangular"):
        E.lsqr(A, b, precond_R=E.DenseMatrix(low))
    sing = np.triu(np.ones((5, 5)))
    sing[2, 2] = 0.0
    with pytest.raises(E.SingularFactorError, match="zero diagonal entry at index 2"):
        E.lsqr(A, b, precond_R=E.DenseMatrix(sing))
    with pytest.raises(E.ShapeError, match="A is 40x5 but b has length 3"):
        E.lsqr(A, E.Vector(np.ones(3)))


def test_solve_rejects_unknown_method_and_defaults_to_lsqr():
    import inspect

    A, b = _prob()
    with pytest.raises(E.SpecError, match="unknown method 'qr'"):
        E.solve(E.LeastSquaresProblem(A=A, b=b), "qr")
    assert inspect.signature(E.solve).parameters["method"].default == "lsqr"
    assert E.METHODS == ("lsqr", "saa", "sap", "direct")
