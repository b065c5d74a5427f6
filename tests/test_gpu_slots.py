"""The reduce of the row-sharded apply (distributed.PeerReduce,
skl_reduce_peers, skl_sum_slots) on one GPU: ranks are emulated as shards
whose partials live in separate buffers (no kernel waits on another), each
emulated rank reduces its element block, and the real symmetric-memory path
runs end to end with a one-rank process group."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_fro

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_14309_b200 as E  # noqa: E402
from paper_2409_14309_b200 import _native  # noqa: E402
from paper_2409_14309_b200.distributed import (  # noqa: E402
    ShardPlan,
    csr_row_block,
    element_block,
    local_partial_device,
    partial_ld,
    shard_rows,
)

ROOT = Path(__file__).resolve().parents[1]


def test_sum_slots_is_the_ordered_fold():
    rng = np.random.default_rng(3)
    nslots, rows, cols = 5, 77, 9
    ld = 78
    stride = ld * cols + 6
    host = rng.standard_normal(nslots * stride) * np.logspace(0, 12, nslots * stride)
    slots = torch.from_numpy(host).cuda()
    out = torch.empty((cols, 80), dtype=torch.float64, device="cuda")
    _native.call("skl_sum_slots", _native.ptr(slots), nslots, stride, rows, cols, ld,
                 _native.ptr(out), 80, torch.cuda.current_stream().cuda_stream)
    want = np.zeros((rows, cols))
    for c in range(cols):
        s = host[c * ld:c * ld + rows].copy()
        for q in range(1, nslots):
            s = s + host[q * stride + c * ld:q * stride + c * ld + rows]
        want[:, c] = s
    got = out.cpu().numpy()[:, :rows].T
    assert got.tobytes() == np.ascontiguousarray(want).tobytes()
    with pytest.raises(E.ShapeError):
        _native.call("skl_sum_slots", _native.ptr(slots), nslots, 10, rows, cols, ld,
                     _native.ptr(out), 80, torch.cuda.current_stream().cuda_stream)


def _reduce_emulated(bufs, total, out):
    """Every emulated rank reduces its element block of the partials into out."""
    world = len(bufs)
    arr = _native.ptr_array([t.data_ptr() for t in bufs])
    for r in range(world):
        e0, e1 = element_block(total, world, r)
        _native.call("skl_reduce_peers", arr, world, e0, e1, out.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("world,total", [(1, 10), (2, 7), (3, 1001), (8, 2 * 4096 + 3),
                                         (16, 64)])
def test_reduce_peers_is_the_ordered_fold(world, total):
    rng = np.random.default_rng(world * 1000 + total)
    host = [rng.standard_normal(total) * 10.0 ** rng.integers(-8, 8, total) for _ in range(world)]
    bufs = [torch.from_numpy(h).cuda() for h in host]
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    _reduce_emulated(bufs, total, out)
    want = host[0].copy()
    for h in host[1:]:
        want = want + h
    assert out.cpu().numpy().tobytes() == want.tobytes()
    # the same bits as the single-buffer slot sum
    if total > 1:
        slots = torch.cat(bufs)
        o2 = torch.empty(total, dtype=torch.float64, device="cuda")
        _native.call("skl_sum_slots", slots.data_ptr(), world, total, total, 1, total,
                     o2.data_ptr(), total, torch.cuda.current_stream().cuda_stream)
        assert torch.equal(o2, out)


def test_reduce_peers_unaligned_and_errors():
    a = torch.arange(11, dtype=torch.float64, device="cuda")
    b = torch.arange(11, dtype=torch.float64, device="cuda") * 3
    out = torch.zeros(12, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    # odd begin and an out pointer off 16 bytes: scalar path
    _native.call("skl_reduce_peers", _native.ptr_array([a.data_ptr() + 8, b.data_ptr() + 8]), 2,
                 1, 9, out.data_ptr() + 8, st)
    got = out.cpu().numpy()
    want = (np.arange(11.0) * 4)[1:10]
    assert np.array_equal(got[2:10], want[1:9]) and got[0] == 0 and got[1] == 0
    with pytest.raises(E.ShapeError):
        _native.call("skl_reduce_peers", _native.ptr_array([a.data_ptr()] * 17), 17, 0, 4,
                     out.data_ptr(), st)


@pytest.mark.parametrize("kind,m,n,d,world,csr", [("countsketch", 60_000, 6, 512, 4, False),
                                                  ("srht", 1 << 16, 3, 256, 2, False),
                                                  ("gaussian", 20_000, 5, 128, 3, False),
                                                  ("countsketch", 100_000, 40, 1024, 4, True),
                                                  ("countsketch", 50_000, 12, 8192, 3, True),
                                                  ("srht", 1 << 15, 7, 64, 2, True)])
def test_emulated_ranks_partials_then_peer_reduce(kind, m, n, d, world, csr):
    """Each 'rank' writes its partial straight into its own buffer (the
    kernels' dest pointer) -- dense or CSR row blocks -- then every rank
    reduces its element block: bitwise the ordered fold of the per-shard
    partials and within 1e-13 of the one-device S[A|b]."""
    import scipy.sparse

    rng = np.random.default_rng(m + world)
    if csr:
        A_sp = scipy.sparse.random(m, n, density=min(1.0, 3.0 / n), format="csr",
                                   random_state=int(m % 1000), data_rvs=rng.standard_normal)
        A_sp.sort_indices()
        A = np.asfortranarray(A_sp.toarray())
    else:
        A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec(kind, d, seed=5), m)
    ld = partial_ld(d)
    slot = (n + 1) * ld
    bufs = [torch.zeros(slot, dtype=torch.float64, device="cuda") for _ in range(world)]
    parts = []
    for r in range(world):
        r0, r1 = shard_rows(m, world, r)
        bd = torch.from_numpy(b[r0:r1].copy()).cuda()
        if csr:
            Al, lda = csr_row_block(A_sp, r0, r1), 0
        else:
            Al, lda = torch.from_numpy(np.asfortranarray(A[r0:r1])).cuda(), r1 - r0
        plan = ShardPlan(op, r0, r1)
        assert local_partial_device(plan, Al, lda, bd, dest=bufs[r].data_ptr()) is None
        parts.append(local_partial_device(plan, Al, lda, bd)[:d].cpu().numpy())
        assert np.array_equal(parts[-1], bufs[r].view(n + 1, ld).t()[:d].cpu().numpy())
    out = torch.empty(slot, dtype=torch.float64, device="cuda")
    _reduce_emulated(bufs, slot, out)
    got = out.view(n + 1, ld).t()[:d].cpu().numpy()
    want = parts[0].copy()
    for p in parts[1:]:
        want = want + p
    assert got.tobytes() == np.ascontiguousarray(want).tobytes()
    Ac = E.SparseMatrix.from_scipy(A_sp) if csr else E.DenseMatrix(A)
    full = np.column_stack([E.apply_to_matrix(op, Ac).data, E.apply_to_vector(op, E.Vector(b)).data])
    assert rel_fro(got, full) <= 1e-13


SCRIPT = r'''
import os, sys, numpy as np, scipy.sparse, torch, torch.distributed as dist
sys.path.insert(0, os.environ["SKL_ROOT"])
import paper_2409_14309_b200 as E
from paper_2409_14309_b200.distributed import PeerReduce, csr_row_block, sharded_sketch_and_apply
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
rng = np.random.default_rng(0)
A = rng.standard_normal((30000, 12)); b = rng.standard_normal(30000)
Ad = torch.from_numpy(np.asfortranarray(A)).cuda(); bd = torch.from_numpy(b).cuda()
spec = E.SketchSpec("countsketch", 96, seed=3)
x, rn, d = sharded_sketch_and_apply(Ad, bd, 30000, spec, dist, collective="peer")
op = E.build_sketch(spec, 30000)
SA = E.apply_to_matrix(op, E.DenseMatrix(A)).data; Sb = E.apply_to_vector(op, E.Vector(b)).data
xw = np.linalg.lstsq(SA, Sb, rcond=None)[0]
assert np.linalg.norm(x.cpu().numpy() - xw) <= 1e-10 * np.linalg.norm(xw), "x mismatch"
assert abs(rn - np.linalg.norm(A @ xw - b)) <= 1e-10 * rn
# CSR row block through the same peer path
S = scipy.sparse.random(40000, 30, density=0.05, format="csr", random_state=1)
S.sort_indices()
bs = rng.standard_normal(40000)
x2, rn2, d2 = sharded_sketch_and_apply(csr_row_block(S, 0, 40000), torch.from_numpy(bs).cuda(),
                                       40000, E.SketchSpec("countsketch", 256, seed=4), dist,
                                       collective="peer")
op2 = E.build_sketch(E.SketchSpec("countsketch", 256, seed=4), 40000)
SA2 = E.apply_to_matrix(op2, E.SparseMatrix.from_scipy(S)).data
Sb2 = E.apply_to_vector(op2, E.Vector(bs)).data
xw2 = np.linalg.lstsq(SA2, Sb2, rcond=None)[0]
assert np.linalg.norm(x2.cpu().numpy() - xw2) <= 1e-10 * np.linalg.norm(xw2), "csr x mismatch"
assert abs(rn2 - np.linalg.norm(S @ xw2 - bs)) <= 1e-10 * rn2
pr = PeerReduce(96, 13)
assert pr.partial_ptr() == pr.buf.data_ptr() and (pr.e0, pr.e1) == (0, 13 * 96)
dist.destroy_process_group()
print("PEER-OK")
'''


def test_peer_reduce_end_to_end_one_rank(tmp_path):
    """The symmetric-memory rendezvous, the kernels' writes into the rank's
    own buffer, the barriers and the peer reduce, through
    sharded_sketch_and_apply with a one-rank NCCL group (dense and CSR row
    blocks; a fresh process: the group is process-global)."""
    script = tmp_path / "peer.py"
    script.write_text(SCRIPT)
    env = dict(os.environ, SKL_ROOT=str(ROOT), MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(29500 + os.getpid() % 1000), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "PEER-OK" in out.stdout, out.stderr[-3000:]
