"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(`sketchls`), runs its public API on seeded inputs from
paper_2409_14309_b200.workloads (numpy backend) and writes
tests/golden/golden.npz.  The fixtures pin (a) the oracle restatement
(tests/test_oracle_golden.py, CPU) and (b) the CUDA engine
(tests/test_gpu_parity.py).  /root/reference is never read at test time.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import scipy
import scipy.sparse

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import sketchls as ref  # noqa: E402
from sketchls.rng import derive_seed, stream  # noqa: E402

from paper_2409_14309_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cs_hashes(op):
    coo = op.sparse_map.tocoo()
    order = np.argsort(coo.col, kind="stable")
    return coo.row[order].astype(np.int32), coo.data[order].astype(np.int8)


def main() -> None:
    g: dict[str, np.ndarray] = {}
    meta: dict[str, object] = {"numpy": np.__version__, "scipy": scipy.__version__}

    # --- seeds (rng.py:27-40)
    seed_cases = [(0, ()), (5, ("countsketch", 100)), (2**64 - 1, ("saa",)), (123, ("srht", 64)),
                  (9, ("A", 3, "noise"))]
    meta["derive_seed"] = [[s, list(t), derive_seed(s, *t)] for s, t in seed_cases]

    # --- CountSketch hashes/signs (sketch.py:97-99)
    for m, d, seed in [(100, 4, 5), (20_000, 800, 0), (4097, 16, 3)]:
        op = ref.build_sketch(ref.SketchSpec("countsketch", d, seed=seed), m)
        rows, signs = cs_hashes(op)
        g[f"cs_rows_{m}_{d}_{seed}"] = rows
        g[f"cs_signs_{m}_{d}_{seed}"] = signs
    for m, d, seed in [(1 << 20, 2048, 7), (1 << 22, 8192, 11)]:
        op = ref.build_sketch(ref.SketchSpec("countsketch", d, seed=seed), m)
        rows, signs = cs_hashes(op)
        meta[f"cs_sha_{m}_{d}_{seed}"] = sha(rows, signs)
        g[f"cs_rows_head_{m}_{d}_{seed}"] = rows[:4096]
        g[f"cs_rows_tail_{m}_{d}_{seed}"] = rows[-4096:]

    # --- SRHT signs and row samples (sketch.py:116-127)
    for m, d, seed in [(50, 16, 2), (1000, 64, 3), (20_000, 800, 4)]:
        op = ref.build_sketch(ref.SketchSpec("srht", d, seed=seed), m)
        g[f"srht_signs_{m}_{d}_{seed}"] = op.sign_diag.astype(np.int8)
        g[f"srht_sample_{m}_{d}_{seed}"] = op.row_sample
        meta[f"srht_pad_{m}_{d}_{seed}"] = op.padded_dim
    op = ref.build_sketch(ref.SketchSpec("srht", 2048, seed=5), 1 << 20)
    meta["srht_sha_1048576_2048_5"] = sha(op.sign_diag.astype(np.int8))
    g["srht_sample_1048576_2048_5"] = op.row_sample

    # --- Gaussian entries (sketch.py:94-96)
    op = ref.build_sketch(ref.SketchSpec("gaussian", 16, seed=1), 64)
    g["gauss_16_64_1"] = op.gaussian_entries
    op = ref.build_sketch(ref.SketchSpec("gaussian", 2048, seed=3), 262_144)
    G = op.gaussian_entries
    g["gauss_cfg3_head"] = G.ravel()[:4096].copy()
    g["gauss_cfg3_tail"] = G.ravel()[-4096:].copy()
    g["gauss_cfg3_rowsums"] = G.sum(axis=1)
    del G, op

    # --- FWHT known answers (test_sketch.py:29-36)
    for i, v in enumerate(([1.0, 0, 0, 0], [1.0, 1, 1, 1], [1.0, 2, 3, 4])):
        g[f"fwht_in_{i}"] = np.array(v)
        g[f"fwht_out_{i}"] = ref.fwht_inplace(np.array(v))
    x = stream(4).standard_normal((1024, 3))
    g["fwht_in_1024x3"] = x
    g["fwht_out_1024x3"] = ref.fwht_inplace(x.copy())

    # --- small applies of every engine kind (test_sketch.py:159-166 shapes)
    a = stream(7).standard_normal((64, 5))
    g["small_A"] = a
    for kind in ("gaussian", "srht", "countsketch", "identity"):
        op = ref.build_sketch(ref.SketchSpec(kind, 16, seed=42), 64)
        g[f"small_SA_{kind}"] = ref.apply_to_matrix(op, ref.DenseMatrix(a)).data
        g[f"small_Sb_{kind}"] = ref.apply_to_vector(op, ref.Vector(a[:, 0].copy())).data

    # --- QR conventions (linalg.py:166-192)
    for m, n, seed in [(5, 3, 0), (20, 5, 1), (100, 40, 2)]:
        M = stream(seed).standard_normal((m, n))
        f = ref.economy_qr(ref.DenseMatrix(M))
        g[f"qr_M_{m}_{n}"] = M
        g[f"qr_Q_{m}_{n}"] = f.Q.data
        g[f"qr_R_{m}_{n}"] = f.R.data

    # --- SAA solves on the configs (full cfg1, reduced cfg2-5)
    saa_cases = {
        "cfg1": (W.config(1), "countsketch"),
        "cfg2r": (W.config(2, m=1 << 14), "countsketch"),
        "cfg3r": (W.config(3, m=8192, n=64, d=256), "gaussian"),
        "cfg4r": (W.config(4, m=1 << 16, n=256, d=2048), "countsketch"),
        "cfg5r": (W.config(5, m=6000, n=32, d=256), "srht"),
        "cfg5r_cs": (W.config(5, m=6000, n=32, d=256), "countsketch"),
    }
    for name, (c, kind) in saa_cases.items():
        A, b, _ = W.make_problem(c)
        Ac = ref.SparseMatrix.from_scipy(A) if scipy.sparse.issparse(A) else ref.DenseMatrix(A)
        prob = ref.LeastSquaresProblem(A=Ac, b=ref.Vector(b))
        spec = ref.SketchSpec(kind, 1, seed=W.SEED)
        opts = ref.SolverOptions(d_factor=c.d / c.n)
        res = ref.solve(prob, "saa", spec, opts)
        assert res.d == c.d, (name, res.d, c.d)
        op = ref.build_sketch(ref.SketchSpec(kind, c.d, seed=derive_seed(W.SEED, "saa")), c.m)
        SA = ref.apply_to_matrix(op, Ac).data
        Sb = ref.apply_to_vector(op, ref.Vector(b)).data
        g[f"{name}_x"] = res.x.data
        g[f"{name}_Sb"] = Sb
        meta[f"{name}_residual"] = res.residual_norm
        meta[f"{name}_SA_sha"] = sha(np.asfortranarray(SA))
        meta[f"{name}_SA_fro"] = float(np.linalg.norm(SA))
        if SA.size <= 300_000:
            g[f"{name}_SA"] = SA
        else:
            g[f"{name}_SA_cols"] = SA[:, :4].copy()
        meta[f"{name}_shape"] = [c.m, c.n, c.d]

    # --- sparse sign embeddings (sketch.py:104-115, 130-149): both row-sampling
    # regimes (argpartition when d <= 4 s^2, integers + redraw otherwise)
    for m, d, s_, seed in [(60, 32, 5, 5), (40, 9, 8, 1), (3000, 64, 8, 2), (5000, 2048, 8, 3),
                           (20_000, 800, 8, 4), (100, 8, 8, 6)]:
        op = ref.build_sketch(ref.SketchSpec("sparsesign", d, seed=seed, sparsity=s_), m)
        coo = op.sparse_map.tocoo()
        g[f"ss_row_{m}_{d}_{s_}_{seed}"] = coo.row.astype(np.int32)
        g[f"ss_col_{m}_{d}_{s_}_{seed}"] = coo.col.astype(np.int32)
        g[f"ss_val_{m}_{d}_{s_}_{seed}"] = coo.data
    c = W.config(1)
    A, b, _ = W.make_problem(c)
    prob = ref.LeastSquaresProblem(A=ref.DenseMatrix(A), b=ref.Vector(b))
    res = ref.solve(prob, "saa", ref.SketchSpec("sparsesign", 1, seed=W.SEED),
                    ref.SolverOptions(d_factor=c.d / c.n))
    g["ss_cfg1_x"] = res.x.data
    meta["ss_cfg1_residual"] = res.residual_norm
    op = ref.build_sketch(ref.SketchSpec("sparsesign", c.d, seed=derive_seed(W.SEED, "saa")), c.m)
    meta["ss_cfg1_SA_sha"] = sha(np.asfortranarray(ref.apply_to_matrix(op, ref.DenseMatrix(A)).data))

    # --- SAP (sketch-and-precondition + LSQR, solvers.py:323-361, 110-255)
    sap_cases = {
        "sap_cfg1": (W.config(1), "countsketch", True),
        "sap_cfg2r": (W.config(2, m=1 << 14), "countsketch", True),
        "sap_cfg3r": (W.config(3, m=8192, n=64, d=256), "gaussian", True),
        "sap_cfg4r": (W.config(4, m=1 << 16, n=256, d=2048), "countsketch", True),
        "sap_cfg5r": (W.config(5, m=6000, n=32, d=256), "srht", False),
    }
    for name, (c, kind, warm) in sap_cases.items():
        A, b, _ = W.make_problem(c)
        Ac = ref.SparseMatrix.from_scipy(A) if scipy.sparse.issparse(A) else ref.DenseMatrix(A)
        prob = ref.LeastSquaresProblem(A=Ac, b=ref.Vector(b))
        spec = ref.SketchSpec(kind, 1, seed=W.SEED)
        opts = ref.SolverOptions(d_factor=c.d / c.n, warm_start=warm)
        res = ref.solve(prob, "sap", spec, opts)
        assert res.d == c.d, (name, res.d, c.d)
        g[f"{name}_x"] = res.x.data
        meta[f"{name}_residual"] = res.residual_norm
        meta[f"{name}_iterations"] = res.iterations
        meta[f"{name}_termination"] = res.termination
        meta[f"{name}_warm"] = warm
    # plain LSQR (method "lsqr") on a small problem
    c = W.config(1, m=3000, n=40)
    A, b, _ = W.make_problem(c)
    res = ref.solve(ref.LeastSquaresProblem(A=ref.DenseMatrix(A), b=ref.Vector(b)), "lsqr")
    g["lsqr_small_x"] = res.x.data
    meta["lsqr_small_residual"] = res.residual_norm
    meta["lsqr_small_iterations"] = res.iterations
    meta["lsqr_small_termination"] = res.termination

    # --- rank-deficient sketch message (test_solvers.py:121-127)
    rng = stream(15)
    a = rng.standard_normal((50, 4))
    a[:, 3] = a[:, 0]
    bb = rng.standard_normal(50)
    g["rankdef_A"] = a
    g["rankdef_b"] = bb
    try:
        ref.sketch_and_apply(ref.LeastSquaresProblem(A=ref.DenseMatrix(a), b=ref.Vector(bb)),
                             ref.SketchSpec("countsketch", 1, seed=16))
        meta["rankdef_msg"] = None
    except ref.SingularFactorError as exc:
        meta["rankdef_msg"] = str(exc)

    # --- device problem generator (probgen.py:43-80), SURVEY.md §8f f3
    pg_cases = {"pg_tall": (300, 12, 1e6, 1e-4, 3), "pg_square": (40, 40, 1e3, 0.0, 1),
                "pg_col": (50, 1, 1e10, 1e-10, 7), "pg_default": (513, 33, 1e10, 1e-10, 0)}
    for name, (m, n, kappa, beta, seed) in pg_cases.items():
        prob = ref.generate_problem(ref.ProblemSpec(m=m, n=n, kappa=kappa, beta=beta, seed=seed))
        g[f"{name}_A"] = prob.A.data
        g[f"{name}_b"] = prob.b.data
        g[f"{name}_xstar"] = prob.x_star.data
        meta[f"{name}_spec"] = [m, n, kappa, beta, seed]
    # the "direct" method (solvers.py:381-396) on the plain-LSQR problem
    c = W.config(1, m=3000, n=40)
    A, b, _ = W.make_problem(c)
    res = ref.solve(ref.LeastSquaresProblem(A=ref.DenseMatrix(A), b=ref.Vector(b)), "direct")
    g["direct_small_x"] = res.x.data
    meta["direct_small_residual"] = res.residual_norm

    # --- Matrix Market / CLI files written by the reference (mmio.py, probgen.py:83-98,
    # bench.py:186-245), compared byte for byte by tests/test_io_cpu.py
    io = OUT.parent / "io"
    io.mkdir(exist_ok=True)
    dense = np.array([[0.1, -2.5e-7], [1e16, 5e-324], [-0.0, 123456789.0], [1.0 / 3.0, -7.0]])
    ref.write_matrix(str(io / "dense.mtx"), ref.DenseMatrix(dense))
    sp = scipy.sparse.csr_matrix(np.array([[0.0, 1.5, 0.0], [0.0, 0.0, 0.0], [-2.0, 0.0, 1e-300],
                                           [0.0, 3.25, 0.0]]))
    ref.write_matrix(str(io / "sparse.mtx"), ref.SparseMatrix.from_scipy(sp))
    ref.write_vector(str(io / "vector.mtx"), ref.Vector(np.array([2.0, -0.5, 1e-9])))
    (io / "dups.mtx").write_text("%%MatrixMarket matrix coordinate integer general\n"
                                 "% comment line\n3 2 5\n3 1 4\n1 2 1\n3 1 -1\n2 2 7\n1 2 2\n")
    dup = ref.read_matrix(str(io / "dups.mtx"))
    g["io_dups_indptr"], g["io_dups_indices"], g["io_dups_values"] = (
        dup.indptr, dup.indices, dup.values)
    spec = ref.ProblemSpec(m=30, n=4, kappa=1e4, beta=1e-6, seed=11)
    ref.write_problem_dir(spec, ref.generate_problem(spec), str(io / "problem"))

    g["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
