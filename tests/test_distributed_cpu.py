"""Multi-rank row sharding on CPU (gloo, world_size 2).

Exercises the host-side logic of paper_2409_14309_b200.distributed -- shard
boundaries, per-rank slices of the global operator, the reduce of the
d x (n+1) partials, broadcast of x and the residual all-reduce -- with the
per-rank compute supplied by the CPU oracle (the CUDA kernels need a GPU;
their parity is covered by tests/test_gpu_parity.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2409_14309_b200 import SketchSpec, build_sketch
from paper_2409_14309_b200.distributed import ShardPlan, shard_rows, sharded_sketch_and_apply
from paper_2409_14309_b200.sketch import SHARD_ALIGN


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(m, n, seed=5):
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = A @ rng.standard_normal(n) + 1e-3 * rng.standard_normal(m)
    return A, b


def _oracle_partial(plan, A_local, b_local):
    a = A_local.numpy()
    bb = b_local.numpy()
    rows, signs = plan.rows.astype(np.int64), plan.signs.astype(np.float64)
    SA = O.countsketch_apply(rows, signs, plan.d, a)
    Sb = O.countsketch_apply(rows, signs, plan.d, bb)
    return torch.from_numpy(np.asfortranarray(np.column_stack([SA, Sb])))


def _oracle_partial_any(plan, A_local, b_local):
    """S[:, r0:r1] [A_local | b_local] for any kind: the global operator
    applied to the full-height matrix that is zero outside the shard."""
    m = plan.op.source_dim
    key = O.derive_seed(plan.op_seed, plan.kind, m)
    a = np.zeros((m, A_local.shape[1]))
    a[plan.r0:plan.r1] = A_local.numpy()
    bb = np.zeros(m)
    bb[plan.r0:plan.r1] = b_local.numpy()
    SA, Sb = O.sketch_apply(plan.kind, key, plan.d, a, bb)
    return torch.from_numpy(np.asfortranarray(np.column_stack([SA, Sb])))


def _oracle_solve(partial):
    p = partial.numpy()
    q, r = O.economy_qr(p[:, :-1])
    import scipy.linalg

    x = scipy.linalg.solve_triangular(r, q.T @ p[:, -1], lower=False)
    return torch.from_numpy(x)


def _oracle_r2(A_local, b_local, x):
    r = A_local.numpy() @ x.numpy() - b_local.numpy()
    return torch.tensor([float(r @ r)], dtype=torch.float64)


def _worker(rank, world, port, m, n, d, seed, out, kind="countsketch"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, b = _problem(m, n)
        r0, r1 = shard_rows(m, world, rank)
        spec = SketchSpec(kind, d, seed=seed)

        def local(plan, A_local, b_local):
            if kind == "countsketch":
                return _oracle_partial(plan, A_local, b_local)
            plan.op_seed = seed
            return _oracle_partial_any(plan, A_local, b_local)

        x, rnorm, dd = sharded_sketch_and_apply(
            torch.from_numpy(np.asfortranarray(A[r0:r1])), torch.from_numpy(b[r0:r1].copy()), m,
            spec, dist, local_apply=local, solve_reduced=_oracle_solve,
            residual_local=_oracle_r2)
        out[rank] = (x.numpy().copy(), rnorm, dd)
    finally:
        dist.destroy_process_group()


def test_shard_rows_cover_and_align():
    for m in (1, 2047, 2048, 2049, 10_000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            assert all(s0 % SHARD_ALIGN == 0 for s0, _ in spans)


def test_shard_plan_slices_global_hashes():
    op = build_sketch(SketchSpec("countsketch", 64, seed=3), 10_000)
    plan = ShardPlan(op, 4096, 8192)
    assert np.array_equal(plan.rows, op.rows[4096:8192])
    assert np.array_equal(plan.signs, op.signs[4096:8192])


def test_partials_sum_to_global_sketch():
    m, n, d = 9000, 5, 64
    A, b = _problem(m, n)
    op = build_sketch(SketchSpec("countsketch", d, seed=11), m)
    total = 0
    for rank in range(3):
        r0, r1 = shard_rows(m, 3, rank)
        total = total + _oracle_partial(ShardPlan(op, r0, r1), torch.from_numpy(A[r0:r1]),
                                        torch.from_numpy(b[r0:r1].copy())).numpy()
    full = O.countsketch_apply(op.rows.astype(np.int64), op.signs.astype(np.float64), d, A)
    assert np.linalg.norm(total[:, :n] - full) <= 1e-15 * np.linalg.norm(full)


@pytest.mark.timeout(300)
def test_gloo_world2_matches_single_process():
    m, n, d, seed = 8192, 6, 96, 21
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, m, n, d, seed, out), nprocs=2, join=True)
    A, b = _problem(m, n)
    key = O.derive_seed(seed, "countsketch", m)
    rows, signs = O.countsketch_draws(key, m, d)
    SA = O.countsketch_apply(rows, signs, d, A)
    Sb = O.countsketch_apply(rows, signs, d, b)
    q, r = O.economy_qr(SA)
    import scipy.linalg

    x_ref = scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False)
    r_ref = np.linalg.norm(A @ x_ref - b)
    for rank in range(2):
        x, rnorm, dd = out[rank]
        assert dd == d
        assert np.linalg.norm(x - x_ref) <= 1e-12 * np.linalg.norm(x_ref)
        assert abs(rnorm - r_ref) <= 1e-12 * r_ref


@pytest.mark.timeout(300)
@pytest.mark.parametrize("kind", ["srht", "gaussian"])
def test_gloo_world2_other_kinds(kind):
    """SRHT (block-offset sign) and Gaussian (column block) shard plans over
    gloo: the reduced partials solve to the single-process SAA answer."""
    m, n, d, seed = 20_000, 5, 64, 8
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, m, n, d, seed, out, kind), nprocs=2, join=True)
    A, b = _problem(m, n)
    SA, Sb = O.sketch_apply(kind, O.derive_seed(seed, kind, m), d, A, b)
    q, r = O.economy_qr(SA)
    import scipy.linalg

    want = scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False)
    for rank in range(2):
        x, rnorm, dd = out[rank]
        assert dd == d
        assert np.linalg.norm(x - want) <= 1e-10 * np.linalg.norm(want)
        assert abs(rnorm - np.linalg.norm(A @ want - b)) <= 1e-10 * rnorm


def test_srht_shard_must_be_block_aligned():
    op = build_sketch(SketchSpec("srht", 64, seed=1), 20_000)
    with pytest.raises(ValueError):
        ShardPlan(op, 100, 20_000)


def test_element_blocks_tile_and_align():
    """PeerReduce's reduce-scatter split (host logic): the ranks' element
    blocks tile the partial exactly, start 16-byte aligned and are near-equal."""
    from paper_2409_14309_b200.distributed import element_block, partial_ld

    for total in (1, 2, 7, 96 * 13, 8192 * 1025, 2048 * 257):
        for world in (1, 2, 3, 8, 16):
            spans = [element_block(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            assert all(e0 % 2 == 0 for e0, _ in spans)
            sizes = [e1 - e0 for e0, e1 in spans]
            assert max(sizes) - min(sizes) <= 2 or total < 2 * world
    assert partial_ld(100) == 100 and partial_ld(101) == 102


def _csr_problem(m, n, seed=3):
    import scipy.sparse

    rng = np.random.default_rng(seed)
    A = scipy.sparse.random(m, n, density=0.02, format="csr", random_state=seed,
                            data_rvs=rng.standard_normal)
    A.sort_indices()
    b = A @ rng.standard_normal(n) + 1e-3 * rng.standard_normal(m)
    return A, b


def _csr_worker(rank, world, port, m, n, d, seed, out):
    import scipy.sparse

    from paper_2409_14309_b200.distributed import csr_row_block

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, b = _csr_problem(m, n)
        r0, r1 = shard_rows(m, world, rank)
        blk = csr_row_block(A, r0, r1, device="cpu")
        assert blk.shape == (r1 - r0, n) and int(blk.indptr[0]) == 0
        assert blk.nnz == int(A.indptr[r1] - A.indptr[r0])

        def to_sp(block):
            return scipy.sparse.csr_matrix((block.values.numpy(), block.indices.numpy(),
                                            block.indptr.numpy()), shape=block.shape)

        def local(plan, A_local, b_local):
            rows, signs = plan.rows.astype(np.int64), plan.signs.astype(np.float64)
            SA = O.countsketch_apply(rows, signs, plan.d, to_sp(A_local))
            Sb = O.countsketch_apply(rows, signs, plan.d, b_local.numpy())
            return torch.from_numpy(np.asfortranarray(np.column_stack([SA, Sb])))

        def r2(A_local, b_local, x):
            r = to_sp(A_local) @ x.numpy() - b_local.numpy()
            return torch.tensor([float(r @ r)], dtype=torch.float64)

        x, rnorm, dd = sharded_sketch_and_apply(
            blk, torch.from_numpy(b[r0:r1].copy()), m, SketchSpec("countsketch", d, seed=seed),
            dist, local_apply=local, solve_reduced=_oracle_solve, residual_local=r2)
        out[rank] = (x.numpy().copy(), rnorm, dd)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_csr_row_blocks():
    """CSR row sharding (config 4's layout): each rank holds rows [r0, r1) of
    the CSR with a rebased indptr and sketches them with the global hashes of
    those rows; the reduced partials solve to the single-process answer."""
    m, n, d, seed = 30_000, 40, 256, 9
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_csr_worker, args=(2, port, m, n, d, seed, out), nprocs=2, join=True)
    A, b = _csr_problem(m, n)
    rows, signs = O.countsketch_draws(O.derive_seed(seed, "countsketch", m), m, d)
    SA = O.countsketch_apply(rows, signs, d, A)
    Sb = O.countsketch_apply(rows, signs, d, b)
    q, r = O.economy_qr(SA)
    import scipy.linalg

    x_ref = scipy.linalg.solve_triangular(r, q.T @ Sb, lower=False)
    r_ref = np.linalg.norm(A @ x_ref - b)
    for rank in range(2):
        x, rnorm, dd = out[rank]
        assert dd == d
        assert np.linalg.norm(x - x_ref) <= 1e-12 * np.linalg.norm(x_ref)
        assert abs(rnorm - r_ref) <= 1e-12 * r_ref


def test_band_pieces_tile_every_block():
    """The rectangles a band of normals contributes to a column block: over
    all bands they tile every block exactly once (host logic of the banded
    Gaussian generation, multidevice.py / distributed.py)."""
    from paper_2409_14309_b200.distributed import band_pieces

    rng = np.random.default_rng(0)
    for d, m in [(3, 10), (16, 8192 * 3), (7, 1001)]:
        N = d * m
        for nb in (1, 2, 5):
            cuts = np.sort(rng.integers(0, N + 1, nb - 1))
            ts = list(zip([0, *cuts], [*cuts, N]))
            for r0, r1 in [(0, m), (0, m // 3), (m // 3, m), (m // 2, m // 2 + 1)]:
                cover = np.zeros((d, m), dtype=np.int64)
                for t0, t1 in ts:
                    for ia, ib, a, c in band_pieces(t0, t1, m, r0, r1):
                        assert r0 <= a < c <= r1 and 0 <= ia < ib <= d
                        cover[ia:ib, a:c] += 1
                        # every covered cell's normal index lies in the band
                        tt = np.arange(ia, ib)[:, None] * m + np.arange(a, c)[None, :]
                        assert tt.min() >= t0 and tt.max() < t1
                assert np.all(cover[:, r0:r1] == 1) and cover.sum() == d * (r1 - r0)


def _band_worker(rank, world, port, d, m, cuts, out):
    from paper_2409_14309_b200.distributed import exchange_gaussian_bands

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G = np.random.default_rng(5).standard_normal((d, m))
        ts = list(zip([0, *cuts], [*cuts, d * m]))
        t0, t1 = ts[rank]
        band = None
        if t1 > t0:
            r_lo, r_hi = t0 // m, (t1 - 1) // m + 1
            ldg = m + 3  # any leading dimension
            band = torch.full((r_hi - r_lo, ldg), float("nan"), dtype=torch.float64)
            flat = G.reshape(-1)
            for t in range(t0, t1):  # only the band's own normals are valid
                band[t // m - r_lo, t % m] = flat[t]
        spans = [shard_rows(m, world, k) for k in range(world)]
        blk, ldb = exchange_gaussian_bands(band, t0, t1, ts, m, d, spans, rank, dist)
        r0, r1 = spans[rank]
        out[rank] = (blk[:, : r1 - r0].numpy().copy(), G[:, r0:r1].copy(), ldb)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world3_gaussian_band_exchange():
    """The all-to-all of the banded Gaussian generation (distributed.py):
    ranks holding arbitrary bands of the d x m operator's normals end with
    exactly their column blocks (bands cut mid-row, one empty band)."""
    d, m, world = 6, 3 * 8192, 3
    N = d * m
    cuts = [N // 3 + 17, N // 3 + 17]  # rank 1's band is empty
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_band_worker, args=(world, port, d, m, cuts, out), nprocs=world, join=True)
    for rank in range(world):
        got, want, ldb = out[rank]
        assert np.array_equal(got, want) and ldb % 32 == 0
