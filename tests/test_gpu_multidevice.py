"""solve() over a device list (SolverOptions.devices, multidevice.py) and the
stream safety of the operator's device caches.  One GPU: a device repeated
in the list runs the N-shard logic (row blocks, per-shard plans, fixed-order
reduce, per-block residuals) as separate shards on that device."""

import threading

import numpy as np
import pytest
import scipy.sparse

from conftest import rel_fro

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2409_14309_b200 as E  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _dense(m, n, seed):
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = A @ rng.standard_normal(n) + 1e-3 * rng.standard_normal(m)
    return A, b


@pytest.mark.parametrize("kind,m,n,d_factor,devices", [
    ("countsketch", 100_000, 20, 8, (0, 0, 0, 0)),
    ("countsketch", 1 << 18, 64, 4, (0, 0)),
    ("srht", 1 << 16, 16, 8, (0, 0, 0)),
    ("gaussian", 70_000, 12, 4, (0, 0, 0, 0, 0, 0, 0, 0)),
])
@pytest.mark.parametrize("on_device", [False, True])
def test_solve_over_device_list_matches_oracle(kind, m, n, d_factor, devices, on_device):
    A, b = _dense(m, n, m + n)
    Ac = E.DenseMatrix(torch.from_numpy(A).cuda()) if on_device else E.DenseMatrix(A)
    bc = E.Vector(torch.from_numpy(b).cuda()) if on_device else E.Vector(b)
    spec = E.SketchSpec(kind, 1, seed=17)
    res = E.solve(E.LeastSquaresProblem(Ac, bc), "saa", spec,
                  E.SolverOptions(d_factor=d_factor, devices=devices))
    one = E.solve(E.LeastSquaresProblem(Ac, bc), "saa", spec, E.SolverOptions(d_factor=d_factor))
    want = O.saa_solve(A, b, kind, 17, d_factor)
    x = res.x.data.cpu().numpy() if on_device else res.x.data
    assert res.d == want["d"] == one.d and res.method == "saa" and res.sketch == kind
    assert rel_fro(x, want["x"]) <= 1e-11
    assert abs(res.residual_norm - want["residual"]) <= 1e-11 * want["residual"]
    x1 = one.x.data.cpu().numpy() if on_device else one.x.data
    assert rel_fro(x, x1) <= 1e-12


def test_solve_over_device_list_csr():
    rng = np.random.default_rng(4)
    m, n = 200_000, 64
    S = scipy.sparse.random(m, n, density=0.03, format="csr", random_state=4,
                            data_rvs=rng.standard_normal)
    S.sort_indices()
    b = S @ rng.standard_normal(n) + 1e-3 * rng.standard_normal(m)
    prob = E.LeastSquaresProblem(E.SparseMatrix.from_scipy(S), E.Vector(b))
    spec = E.SketchSpec("countsketch", 1, seed=5)
    res = E.solve(prob, "saa", spec, E.SolverOptions(d_factor=8, devices=(0, 0, 0)))
    want = O.saa_solve(S, b, "countsketch", 5, 8)
    assert rel_fro(res.x.data, want["x"]) <= 1e-11
    assert abs(res.residual_norm - want["residual"]) <= 1e-11 * want["residual"]


def test_single_entry_device_list_is_the_one_device_path():
    A, b = _dense(30_000, 10, 1)
    prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
    spec = E.SketchSpec("countsketch", 1, seed=2)
    r1 = E.solve(prob, "saa", spec, E.SolverOptions(d_factor=4, devices=(0,)))
    r0 = E.solve(prob, "saa", spec, E.SolverOptions(d_factor=4))
    assert np.array_equal(r1.x.data, r0.x.data) and r1.residual_norm == r0.residual_norm


def test_device_list_errors():
    A, b = _dense(30_000, 10, 1)
    prob = E.LeastSquaresProblem(E.DenseMatrix(A), E.Vector(b))
    with pytest.raises(E.SpecError, match="out of range"):
        E.SolverOptions(devices=(0, torch.cuda.device_count()))
    with pytest.raises(E.SpecError, match="nonempty"):
        E.SolverOptions(devices=())
    with pytest.raises(E.SpecError, match="multi-device sketching supports"):
        E.solve(prob, "saa", E.SketchSpec("sparsesign", 1, seed=2),
                E.SolverOptions(d_factor=4, devices=(0, 0)))
    # fewer than 8192 rows per device: the first devices only, same answer
    p9 = E.LeastSquaresProblem(E.DenseMatrix(A[:9000]), E.Vector(b[:9000]))
    r3 = E.solve(p9, "saa", E.SketchSpec("countsketch", 1), E.SolverOptions(d_factor=4,
                                                                          devices=(0, 0, 0)))
    r1 = E.solve(p9, "saa", E.SketchSpec("countsketch", 1), E.SolverOptions(d_factor=4))
    assert rel_fro(r3.x.data, r1.x.data) <= 1e-12


def test_cached_operator_is_safe_across_streams():
    """An operator whose device hashes are still being drawn on one stream is
    handed to a caller on another stream: the consumer waits on the build's
    event, so the apply sees the finished hashes."""
    m, n, d = 1 << 20, 4, 2048
    A = torch.from_numpy(np.asfortranarray(np.random.default_rng(0).standard_normal((m, n)))).cuda()
    want = None
    for trial in range(3):
        E.clear_operator_cache()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        spec = E.SketchSpec("countsketch", d, seed=100 + trial)
        with torch.cuda.stream(s1):
            torch.cuda._sleep(50_000_000)  # keep s1 busy: the draw queues behind it
            op = E.build_sketch(spec, m)
        with torch.cuda.stream(s2):
            SA = E.apply_to_matrix(op, E.DenseMatrix(A)).data
        got = SA.cpu().numpy()
        rows, signs = O.countsketch_draws(O.derive_seed(100 + trial, "countsketch", m), m, d)
        want = O.countsketch_apply(rows, signs, d, A.cpu().numpy())
        assert np.array_equal(got, want)


def test_concurrent_first_use_from_threads():
    """Several threads, each on its own stream, use one fresh operator at
    once: one build, every result bitwise the oracle's."""
    m, n, d = 300_000, 8, 1024
    A_h = np.asfortranarray(np.random.default_rng(1).standard_normal((m, n)))
    A = torch.from_numpy(A_h).cuda()
    E.clear_operator_cache()
    op = E.build_sketch(E.SketchSpec("countsketch", d, seed=3), m)
    rows, signs = O.countsketch_draws(O.derive_seed(3, "countsketch", m), m, d)
    want = O.countsketch_apply(rows, signs, d, A_h)
    out, errs = {}, []

    def work(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[i] = E.apply_to_matrix(op, E.DenseMatrix(A)).data.cpu().numpy()
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for i in range(4):
        assert np.array_equal(out[i], want)


@pytest.mark.parametrize("d,m,world", [(64, 50_000, 8), (16, 3 * 8192, 3), (300, 70_001, 5),
                                       (2048, 262_144, 8)])
def test_gaussian_bands_equal_one_device_operator(d, m, world):
    """Banded generation over a device list (each 'device' parses ~1/N of the
    ziggurat stream, then the bands are exchanged into column blocks): every
    block is bitwise the one-device G[:, r0:r1] -- including config 3's
    2048 x 262144 operator."""
    from paper_2409_14309_b200.distributed import shard_rows
    from paper_2409_14309_b200.multidevice import gaussian_column_blocks

    op = E.build_sketch(E.SketchSpec("gaussian", d, seed=d + m), m)
    spans = [shard_rows(m, world, k) for k in range(world)]
    blocks = gaussian_column_blocks(op, (0,) * world, spans)
    G, _ = op.device_gaussian()
    for (r0, r1), (blk, ldb) in zip(spans, blocks):
        assert ldb >= r1 - r0
        assert torch.equal(blk[:, : r1 - r0], G[:, r0:r1])
