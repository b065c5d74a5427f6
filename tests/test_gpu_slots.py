"""The fused reduce of the row-sharded apply (distributed.PeerSlots,
skl_sum_slots) on one GPU: ranks are emulated as shards written into the
slots of one buffer (no kernel waits on another), and the real symmetric-
memory path runs end to end with a one-rank process group."""

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


@pytest.mark.parametrize("kind,m,n,d,world", [("countsketch", 60_000, 6, 512, 4),
                                              ("srht", 1 << 16, 3, 256, 2),
                                              ("gaussian", 20_000, 5, 128, 3)])
def test_emulated_ranks_write_slots_then_fixed_order_sum(kind, m, n, d, world):
    """Each 'rank' writes its partial straight into its slot (the kernels'
    dest pointer), then one fixed-order sum -- bitwise the ordered fold of the
    per-shard partials and within 1e-13 of the one-device S[A|b]."""
    rng = np.random.default_rng(m + world)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    op = E.build_sketch(E.SketchSpec(kind, d, seed=5), m)
    ld = partial_ld(d)
    slot = (n + 1) * ld
    buf = torch.zeros(world * slot, dtype=torch.float64, device="cuda")
    parts = []
    for r in range(world):
        r0, r1 = shard_rows(m, world, r)
        Ad = torch.from_numpy(np.asfortranarray(A[r0:r1])).cuda()
        bd = torch.from_numpy(b[r0:r1].copy()).cuda()
        plan = ShardPlan(op, r0, r1)
        assert local_partial_device(plan, Ad, r1 - r0, bd, dest=buf.data_ptr() + 8 * r * slot) is None
        parts.append(local_partial_device(plan, Ad, r1 - r0, bd)[:d].cpu().numpy())
    out = torch.empty((n + 1, ld), dtype=torch.float64, device="cuda")
    _native.call("skl_sum_slots", buf.data_ptr(), world, slot, d, n + 1, ld, _native.ptr(out), ld,
                 torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy()[:, :d].T
    want = parts[0].copy()
    for p in parts[1:]:
        want = want + p
    assert got.tobytes() == np.ascontiguousarray(want).tobytes()
    full = np.column_stack([E.apply_to_matrix(op, E.DenseMatrix(A)).data,
                            E.apply_to_vector(op, E.Vector(b)).data])
    assert rel_fro(got, full) <= 1e-13


SCRIPT = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["SKL_ROOT"])
import paper_2409_14309_b200 as E
from paper_2409_14309_b200.distributed import PeerSlots, sharded_sketch_and_apply
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
slots = PeerSlots(96, 13)
p0, p1, p2 = slots.slot_ptr(), (slots.finish(), slots.slot_ptr())[1], (slots.finish(), slots.slot_ptr())[1]
assert p0 == p2 and p1 != p0, "parity double-buffering"
dist.destroy_process_group()
print("PEER-OK")
'''


def test_peer_slots_end_to_end_one_rank(tmp_path):
    """The symmetric-memory rendezvous, the kernels' peer-slot writes, the
    device barrier and the slot sum, through sharded_sketch_and_apply with a
    one-rank NCCL group (a fresh process: the group is process-global)."""
    script = tmp_path / "peer.py"
    script.write_text(SCRIPT)
    env = dict(os.environ, SKL_ROOT=str(ROOT), MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(29500 + os.getpid() % 1000), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "PEER-OK" in out.stdout, out.stderr[-3000:]
