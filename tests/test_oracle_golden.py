"""Pin the CPU oracle (oracle/) against fixtures produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest
import scipy.sparse

from oracle import clib
from oracle import oracle as O
from paper_2409_14309_b200 import workloads as W
from paper_2409_14309_b200._ziggurat import ZIGGURAT_NOR_INV_R, ZIGGURAT_NOR_R, tables

from conftest import rel_fro


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_derive_seed(golden_meta):
    for seed, tags, want in golden_meta["derive_seed"]:
        assert O.derive_seed(seed, *tags) == want


@pytest.mark.parametrize("m,d,seed", [(100, 4, 5), (20_000, 800, 0), (4097, 16, 3)])
def test_countsketch_draws(golden, m, d, seed):
    key = O.derive_seed(seed, "countsketch", m)
    rows, signs = O.countsketch_draws(key, m, d)
    assert np.array_equal(rows, golden[f"cs_rows_{m}_{d}_{seed}"])
    assert np.array_equal(signs, golden[f"cs_signs_{m}_{d}_{seed}"])
    crow, csig = clib.countsketch(key, m, d)
    assert np.array_equal(crow, rows) and np.array_equal(csig, signs)


@pytest.mark.parametrize("m,d,seed", [(1 << 20, 2048, 7), (1 << 22, 8192, 11)])
def test_countsketch_draws_large_digest(golden, golden_meta, m, d, seed):
    key = O.derive_seed(seed, "countsketch", m)
    rows, signs = clib.countsketch(key, m, d)
    assert sha(rows.astype(np.int32), signs.astype(np.int8)) == golden_meta[f"cs_sha_{m}_{d}_{seed}"]
    assert np.array_equal(rows[:4096], golden[f"cs_rows_head_{m}_{d}_{seed}"])
    assert np.array_equal(rows[-4096:], golden[f"cs_rows_tail_{m}_{d}_{seed}"])


def test_lemire_rejection_path_matches_numpy():
    # threshold (2^32 - d) mod d ~ 0.3 * 2^32: every third draw is rejected
    m, d = 4000, 1_500_000_000
    g = O.stream(11)
    want_rows = g.integers(0, d, size=m)
    want_signs = 2.0 * g.integers(0, 2, size=m) - 1.0
    rows, signs = clib.countsketch(11, m, d)
    assert np.array_equal(rows, want_rows) and np.array_equal(signs, want_signs)


def test_u32_stream_matches_numpy():
    key = 0xDEADBEEF12345678
    bg = np.random.Philox(key=key)
    raw = np.array([bg.random_raw() for _ in range(64)], dtype=np.uint64)
    want = np.stack([raw & 0xFFFFFFFF, raw >> 32], axis=1).ravel().astype(np.uint32)
    assert np.array_equal(clib.u32(key, 128), want)


@pytest.mark.parametrize("m,d,seed", [(50, 16, 2), (1000, 64, 3), (20_000, 800, 4)])
def test_srht_draws(golden, golden_meta, m, d, seed):
    key = O.derive_seed(seed, "srht", m)
    signs, sample, m_pad = O.srht_draws(key, m, d)
    assert m_pad == golden_meta[f"srht_pad_{m}_{d}_{seed}"]
    assert np.array_equal(signs.astype(np.int8), golden[f"srht_signs_{m}_{d}_{seed}"])
    assert np.array_equal(sample, golden[f"srht_sample_{m}_{d}_{seed}"])
    cs, cp = clib.srht(key, m_pad, d)
    assert np.array_equal(cs, signs) and np.array_equal(cp, sample)


def test_srht_draws_large(golden, golden_meta):
    key = O.derive_seed(5, "srht", 1 << 20)
    signs, sample = clib.srht(key, 1 << 20, 2048)
    assert sha(signs.astype(np.int8)) == golden_meta["srht_sha_1048576_2048_5"]
    assert np.array_equal(sample, golden["srht_sample_1048576_2048_5"])


def test_gaussian_small(golden):
    key = O.derive_seed(1, "gaussian", 64)
    assert np.array_equal(O.gaussian_draws(key, 16, 64), golden["gauss_16_64_1"])
    ki, wi, fi = tables()
    z = clib.gaussian(key, 16 * 64, ki, wi, fi, ZIGGURAT_NOR_R, ZIGGURAT_NOR_INV_R)
    assert np.array_equal(z.reshape(16, 64) / np.sqrt(16), golden["gauss_16_64_1"])


def test_gaussian_cfg3_head(golden):
    # head of the 2048 x 262144 cfg3 operator: C restatement vs reference
    key = O.derive_seed(3, "gaussian", 262_144)
    ki, wi, fi = tables()
    z = clib.gaussian(key, 4096, ki, wi, fi, ZIGGURAT_NOR_R, ZIGGURAT_NOR_INV_R)
    assert np.array_equal(z / np.sqrt(2048), golden["gauss_cfg3_head"])


def test_ziggurat_tail_paths_match_numpy():
    # many draws so the wedge (exp) and tail (log1p) branches are exercised
    key = 77
    want = O.stream(key).standard_normal(400_000)
    ki, wi, fi = tables()
    got = clib.gaussian(key, want.size, ki, wi, fi, ZIGGURAT_NOR_R, ZIGGURAT_NOR_INV_R)
    assert np.array_equal(got, want)
    assert np.any(np.abs(want) > ZIGGURAT_NOR_R)  # tail samples present


def test_fwht_known_answers(golden):
    for i in range(3):
        x = golden[f"fwht_in_{i}"].copy()
        assert np.array_equal(O.fwht_inplace(x), golden[f"fwht_out_{i}"])
    x = golden["fwht_in_1024x3"].copy()
    assert np.array_equal(O.fwht_inplace(x), golden["fwht_out_1024x3"])


@pytest.mark.parametrize("kind", ["gaussian", "srht", "countsketch"])
def test_small_applies(golden, kind):
    a = golden["small_A"]
    key = O.derive_seed(42, kind, 64)
    SA, Sb = O.sketch_apply(kind, key, 16, a, a[:, 0].copy())
    assert np.array_equal(SA, golden[f"small_SA_{kind}"])
    assert np.array_equal(Sb, golden[f"small_Sb_{kind}"])


def test_countsketch_fold_is_bitwise_csr_matvecs(golden):
    a = W.make_problem(W.config(1))[0]
    key = O.derive_seed(O.derive_seed(W.SEED, "saa"), "countsketch", a.shape[0])
    rows, signs = O.countsketch_draws(key, a.shape[0], 800)
    want = golden["cfg1_SA"]
    assert np.array_equal(O.countsketch_apply(rows, signs, 800, a), want)
    assert np.array_equal(O.countsketch_fold(rows, signs, 800, a), want)
    assert np.array_equal(clib.countsketch_fold(rows, signs, 800, a), want)


@pytest.mark.parametrize("m,n", [(5, 3), (20, 5), (100, 40)])
def test_economy_qr(golden, m, n):
    q, r = O.economy_qr(golden[f"qr_M_{m}_{n}"])
    assert np.array_equal(q, golden[f"qr_Q_{m}_{n}"])
    assert np.array_equal(r, golden[f"qr_R_{m}_{n}"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2r", "cfg3r", "cfg4r", "cfg5r", "cfg5r_cs"])
def test_saa_solves(golden, golden_meta, name):
    m, n, d = golden_meta[f"{name}_shape"]
    cfg = int(name[3])
    kind = "countsketch" if name.endswith("_cs") else W.CONFIGS[cfg].kind
    c = W.config(cfg, m=m, n=n, d=d)
    A, b, _ = W.make_problem(c)
    res = O.saa_solve(A, b, kind, W.SEED, d / n)
    assert res["d"] == d
    assert sha(np.asfortranarray(res["SA"])) == golden_meta[f"{name}_SA_sha"]
    assert np.array_equal(res["Sb"], golden[f"{name}_Sb"])
    assert np.array_equal(res["x"], golden[f"{name}_x"])
    assert res["residual"] == golden_meta[f"{name}_residual"]


def test_rank_deficient_message(golden, golden_meta):
    a, b = golden["rankdef_A"], golden["rankdef_b"]
    key = O.operator_key(16, "countsketch", 50, method="saa")
    SA, _ = O.sketch_apply("countsketch", key, 16, a, b)
    with pytest.raises(O.RankDeficient) as ei:
        O.economy_qr(SA)
    assert f"column {ei.value.col}" in golden_meta["rankdef_msg"]
    assert str(ei.value) in golden_meta["rankdef_msg"]


def test_csr_operand_matches_dense(golden):
    rng = O.stream(8)
    a = np.where(rng.random((64, 6)) < 0.3, rng.standard_normal((64, 6)), 0.0)
    key = O.derive_seed(3, "countsketch", 64)
    rows, signs = O.countsketch_draws(key, 64, 16)
    got = O.countsketch_apply(rows, signs, 16, scipy.sparse.csr_matrix(a))
    assert rel_fro(got, O.countsketch_apply(rows, signs, 16, a)) <= 1e-13


SAP_CASES = {
    "sap_cfg1": (W.config(1), "countsketch"),
    "sap_cfg2r": (W.config(2, m=1 << 14), "countsketch"),
    "sap_cfg3r": (W.config(3, m=8192, n=64, d=256), "gaussian"),
    "sap_cfg4r": (W.config(4, m=1 << 16, n=256, d=2048), "countsketch"),
    "sap_cfg5r": (W.config(5, m=6000, n=32, d=256), "srht"),
}


@pytest.mark.parametrize("name", list(SAP_CASES))
def test_sap_oracle_matches_reference(golden, golden_meta, name):
    """oracle.sap_solve (solvers.py:323-361 + lsqr :110-255) against the
    reference's own solve(problem, "sap", ...) on the same inputs."""
    c, kind = SAP_CASES[name]
    A, b, _ = W.make_problem(c)
    got = O.sap_solve(A, b, kind, W.SEED, c.d / c.n, warm_start=golden_meta[f"{name}_warm"])
    assert got["d"] == c.d
    assert got["iterations"] == golden_meta[f"{name}_iterations"]
    assert got["termination"] == golden_meta[f"{name}_termination"]
    assert rel_fro(got["x"], golden[f"{name}_x"]) <= 1e-12
    assert abs(got["residual"] - golden_meta[f"{name}_residual"]) <= 1e-12 * got["residual"]


def test_plain_lsqr_oracle_matches_reference(golden, golden_meta):
    c = W.config(1, m=3000, n=40)
    A, b, _ = W.make_problem(c)
    got = O.lsqr(np.asfortranarray(A), b)
    assert got["iterations"] == golden_meta["lsqr_small_iterations"]
    assert got["termination"] == golden_meta["lsqr_small_termination"]
    assert rel_fro(got["x"], golden["lsqr_small_x"]) <= 1e-12


SS_CASES = [(60, 32, 5, 5), (40, 9, 8, 1), (3000, 64, 8, 2), (5000, 2048, 8, 3), (20_000, 800, 8, 4),
            (100, 8, 8, 6)]


@pytest.mark.parametrize("m,d,s,seed", SS_CASES)
def test_sparsesign_oracle_structure(golden, m, d, s, seed):
    """oracle.sparsesign_draws/map == the reference's sparse_map (COO triples),
    in both row-sampling regimes (argpartition, integers + redraw) and s == d."""
    rows, signs = O.sparsesign_draws(O.derive_seed(seed, "sparsesign", m), m, d, s)
    coo = O.sparsesign_map(rows, signs, d, m).tocoo()
    assert np.array_equal(coo.row.astype(np.int32), golden[f"ss_row_{m}_{d}_{s}_{seed}"])
    assert np.array_equal(coo.col.astype(np.int32), golden[f"ss_col_{m}_{d}_{s}_{seed}"])
    assert np.array_equal(coo.data, golden[f"ss_val_{m}_{d}_{s}_{seed}"])


@pytest.mark.parametrize("m,d,s,seed", SS_CASES)
def test_sparsesign_engine_draws_match_reference(golden, m, d, s, seed):
    """The engine's operator (numpy draws on the operator stream) builds the
    same S as the reference (CPU: no device needed for the draws)."""
    import paper_2409_14309_b200 as E

    op = E.build_sketch(E.SketchSpec("sparsesign", d, seed=seed, sparsity=s), m)
    coo = op.sparse_map.tocoo()
    assert np.array_equal(coo.row.astype(np.int32), golden[f"ss_row_{m}_{d}_{s}_{seed}"])
    assert np.array_equal(coo.col.astype(np.int32), golden[f"ss_col_{m}_{d}_{s}_{seed}"])
    assert np.array_equal(coo.data, golden[f"ss_val_{m}_{d}_{s}_{seed}"])


def test_sparsesign_saa_oracle(golden, golden_meta):
    c = W.config(1)
    A, b, _ = W.make_problem(c)
    got = O.saa_solve(A, b, "sparsesign", W.SEED, c.d / c.n)
    assert rel_fro(got["x"], golden["ss_cfg1_x"]) <= 1e-12
    assert hashlib.sha256(np.asfortranarray(got["SA"]).tobytes()).hexdigest() == \
        golden_meta["ss_cfg1_SA_sha"]
