"""Full-size digests of BASELINE configs 2-5, computed by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_full.py

Imports the unmodified reference package from /root/reference/pkg/src
(`sketchls`) and records SHA-256 digests of every full-size quantity that
does not depend on the host BLAS (so they hold on any CPU): the operators of
the SAA solves (`solve(..., "saa", SketchSpec(kind, 1, SEED))` builds its
operator from derive_seed(SEED, "saa"), solvers.py:279, sketch.py:93) and
the sketches of BLAS-free inputs:

* cfg2: CountSketch hashes/signs, m = 2^20, d = 2048;
* cfg3: the 2048 x 262144 Gaussian entries (sketch.py:94-96);
* cfg4: hashes/signs at m = 2^22, d = 8192, and the reference's S*A and
  S*b of the config's CSR A and b (csr_matmat / csr_matvec; A and b come from
  the numpy generator and scipy's sparse matvec, no BLAS);
* cfg5: CountSketch hashes/signs and the SRHT sign diagonal + row sample at
  m = 2^23, d = 2048, and the reference's CountSketch S*A of A's first 32
  columns (A is pure normals).

Writes tests/golden/golden_full.json; tests/test_gpu_fullsize.py checks the
engine against it on the GPU box (which never reads /root/reference).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import scipy

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import sketchls as ref  # noqa: E402
from sketchls.rng import derive_seed  # noqa: E402

from paper_2409_14309_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden_full.json"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cs_hashes(op):
    coo = op.sparse_map.tocoo()
    order = np.argsort(coo.col, kind="stable")
    return coo.row[order].astype(np.int32), coo.data[order].astype(np.int8)


def saa_op(kind: str, d: int, m: int):
    return ref.build_sketch(ref.SketchSpec(kind, d, seed=derive_seed(W.SEED, "saa")), m)


def main() -> None:
    meta: dict[str, object] = {"numpy": np.__version__, "scipy": scipy.__version__,
                               "seed": W.SEED}
    # cfg2
    c = W.config(2)
    meta["cfg2_cs_sha"] = sha(*cs_hashes(saa_op("countsketch", c.d, c.m)))
    print("cfg2 done", flush=True)
    # cfg3
    c = W.config(3)
    op = saa_op("gaussian", c.d, c.m)
    meta["cfg3_gauss_sha"] = sha(op.gaussian_entries)
    del op
    print("cfg3 done", flush=True)
    # cfg4
    c = W.config(4)
    A, b, _ = W.make_problem(c)
    op = saa_op("countsketch", c.d, c.m)
    meta["cfg4_cs_sha"] = sha(*cs_hashes(op))
    meta["cfg4_nnz"] = int(A.nnz)
    meta["cfg4_A_sha"] = sha(A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data)
    meta["cfg4_b_sha"] = sha(b)
    SA = ref.apply_to_matrix(op, ref.SparseMatrix.from_scipy(A)).data
    meta["cfg4_SA_sha"] = sha(np.asfortranarray(SA))
    meta["cfg4_Sb_sha"] = sha(ref.apply_to_vector(op, ref.Vector(b)).data)
    del A, b, op, SA
    print("cfg4 done", flush=True)
    # cfg5
    c = W.config(5)
    op = saa_op("countsketch", c.d, c.m)
    meta["cfg5_cs_sha"] = sha(*cs_hashes(op))
    opr = saa_op("srht", c.d, c.m)
    meta["cfg5_srht_signs_sha"] = sha(opr.sign_diag.astype(np.int8))
    meta["cfg5_srht_sample_sha"] = sha(opr.row_sample)
    del opr
    ncol = 32
    from sketchls.rng import stream

    # the first 32 columns of cfg5's A: A = stream(...).standard_normal((n, m)).T,
    # so column c is row c of the (n, m) draw -- the first 32 * m normals
    Asub = stream(derive_seed(W.SEED, "A", c.cfg)).standard_normal((ncol, c.m)).T
    meta["cfg5_A32_sha"] = sha(np.asfortranarray(Asub))
    SA = ref.apply_to_matrix(op, ref.DenseMatrix(Asub)).data
    meta["cfg5_cs_SA32_sha"] = sha(np.asfortranarray(SA))
    print("cfg5 done", flush=True)
    OUT.write_text(json.dumps(meta, indent=1) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
