"""Matrix Market text exchange.

Same file contract as /root/reference/pkg/src/sketchls/mmio.py:1-141:
``array`` (dense, column-major) and ``coordinate`` (sparse, 1-based)
files, field ``real`` or ``integer``, symmetry ``general``; values written
as Python's shortest round-trip ``repr``, so write -> read is bitwise.
Coordinate input is canonicalised (sorted by (row, col), duplicates summed)
before it becomes a ``SparseMatrix``.  Device carriers are copied to the
host for writing.  Text formatting dominates this path, so it stays on the
host; the GPU gains nothing here.
"""

from __future__ import annotations

import numpy as np

from .errors import ShapeError
from .linalg import DenseMatrix, SparseMatrix, Vector

ARRAY_HEADER = "%%MatrixMarket matrix array real general"
COORD_HEADER = "%%MatrixMarket matrix coordinate real general"


def _emit(path: str, lines) -> None:
    with open(path, "w") as fh:
        fh.write("\n".join(lines))
        fh.write("\n")


def _array_lines(a: np.ndarray):
    rows, cols = a.shape
    yield ARRAY_HEADER
    yield f"{rows} {cols}"
    yield from map(repr, np.asarray(a, dtype=np.float64).ravel(order="F").tolist())


def write_matrix(path: str, mat) -> None:
    """Dense -> ``array``; sparse -> ``coordinate`` (mmio.py:23-28)."""
    if isinstance(mat, SparseMatrix):
        rows = np.repeat(np.arange(mat.rows, dtype=np.int64), np.diff(mat.indptr))
        body = (f"{i} {j} {v!r}" for i, j, v in
                zip((rows + 1).tolist(), (mat.indices + 1).tolist(), mat.values.tolist()))
        _emit(path, [COORD_HEADER, f"{mat.rows} {mat.cols} {mat.nnz}", *body])
    else:
        _emit(path, _array_lines(mat.to_numpy()))


def write_vector(path: str, vec: Vector) -> None:
    """An n x 1 ``array`` file (mmio.py:31-33)."""
    _emit(path, _array_lines(np.asarray(vec.to_numpy()).reshape(-1, 1)))


def _parse(path: str) -> tuple[str, list[str]]:
    with open(path) as fh:
        raw = fh.readlines()
    if not raw or not raw[0].startswith("%%MatrixMarket"):
        raise ValueError(f"{path}: missing %%MatrixMarket header")
    head = raw[0].strip().lower().split()
    if len(head) != 5 or head[1] != "matrix":
        raise ValueError(f"{path}: malformed header {raw[0].strip()!r}")
    layout, field, symmetry = head[2:5]
    if layout not in ("array", "coordinate"):
        raise ValueError(f"{path}: unsupported format {layout!r}")
    if field not in ("real", "integer"):
        raise ValueError(f"{path}: unsupported field {field!r}")
    if symmetry != "general":
        raise ValueError(f"{path}: unsupported symmetry {symmetry!r}")
    body = []
    for ln in raw[1:]:
        ln = ln.strip()
        if ln and not ln.startswith("%"):
            body.append(ln)
    if not body:
        raise ValueError(f"{path}: missing size line")
    return layout, body


def _sizes(path: str, line: str, count: int, what: str) -> list[int]:
    try:
        vals = [int(t) for t in line.split()]
    except ValueError:
        vals = []
    if len(vals) != count:
        raise ValueError(f"{path}: bad {what} size line {line!r}")
    return vals


def _dense(path: str, body: list[str]) -> np.ndarray:
    rows, cols = _sizes(path, body[0], 2, "array")
    if len(body) - 1 != rows * cols:
        raise ValueError(f"{path}: expected {rows * cols} entries, found {len(body) - 1}")
    vals = np.array([float(t) for t in body[1:]], dtype=np.float64)
    return vals.reshape((cols, rows)).T  # column-major order on disk


def _sparse(path: str, body: list[str]) -> SparseMatrix:
    rows, cols, nnz = _sizes(path, body[0], 3, "coordinate")
    if len(body) - 1 != nnz:
        raise ValueError(f"{path}: expected {nnz} entries, found {len(body) - 1}")
    ii = np.empty(nnz, dtype=np.int64)
    jj = np.empty(nnz, dtype=np.int64)
    vv = np.empty(nnz, dtype=np.float64)
    for k, ln in enumerate(body[1:]):
        parts = ln.split()
        if len(parts) != 3:
            raise ValueError(f"{path}: bad coordinate entry {ln!r}")
        ii[k], jj[k], vv[k] = int(parts[0]) - 1, int(parts[1]) - 1, float(parts[2])
    if nnz and (ii.min() < 0 or ii.max() >= rows or jj.min() < 0 or jj.max() >= cols):
        raise ValueError(f"{path}: coordinate indices out of range")
    order = np.lexsort((jj, ii))
    ii, jj, vv = ii[order], jj[order], vv[order]
    if nnz > 1:
        first = np.ones(nnz, dtype=bool)
        first[1:] = (ii[1:] != ii[:-1]) | (jj[1:] != jj[:-1])
        if not first.all():
            # sum duplicates in file order within each (row, col) group
            grp = np.cumsum(first) - 1
            acc = np.zeros(int(grp[-1]) + 1, dtype=np.float64)
            np.add.at(acc, grp, vv)
            ii, jj, vv = ii[first], jj[first], acc
    indptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(ii, minlength=rows), out=indptr[1:])
    return SparseMatrix(rows, cols, indptr, jj, vv)


def read_matrix(path: str):
    """``array`` -> DenseMatrix, ``coordinate`` -> SparseMatrix (mmio.py:75-80)."""
    layout, body = _parse(path)
    return DenseMatrix(_dense(path, body)) if layout == "array" else _sparse(path, body)


def read_vector(path: str) -> Vector:
    """A single-column file as a Vector (mmio.py:83-90)."""
    mat = read_matrix(path)
    if isinstance(mat, SparseMatrix):
        mat = mat.densify()
    if mat.cols != 1:
        raise ShapeError(f"{path}: expected a single-column matrix, got {mat.rows}x{mat.cols}")
    return Vector(mat.data[:, 0])
