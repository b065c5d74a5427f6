"""Host side of the native library (no GPU needed): the C-ABI loads and
exports every symbol include/sketchls_b200.h declares, and the bit-exact
host generator / plan builder agree with the oracle and numpy."""

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import clib
from oracle import oracle as O
from paper_2409_14309_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "sketchls_b200.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skl_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.lib()
    names = header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"declared but not exported: {missing}"
    assert lib.skl_abi_version() >= 1


def test_python_signatures_cover_header():
    bound = set(_native.SIGNATURES)
    for n in header_functions():
        assert n in bound, f"{n} declared in the header but not bound in _native.SIGNATURES"


def test_splitmix_and_derive_seed():
    from paper_2409_14309_b200.rng import derive_seed, splitmix64

    for z in (0, 1, 2**63, 2**64 - 1, 0x1234567890ABCDEF):
        assert _native.lib().skl_splitmix64(z) == splitmix64(z) == O.splitmix64(z)
    assert derive_seed(7, "saa", "countsketch", 123) == O.derive_seed(7, "saa", "countsketch", 123)


@pytest.mark.parametrize("offset,count", [(0, 64), (1, 63), (7, 1000), (12345, 777)])
def test_u32_stream_random_access(offset, count):
    key = 0xC0FFEE
    seq = clib.u32(key, offset + count)
    assert np.array_equal(_native.rng_u32(key, offset, count), seq[offset:])


def test_u64_stream_matches_numpy():
    key = 987654321
    bg = np.random.Philox(key=key)
    want = np.array([bg.random_raw() for _ in range(40)], dtype=np.uint64)
    assert np.array_equal(_native.rng_u64(key, 0, 40), want)
    assert np.array_equal(_native.rng_u64(key, 13, 27), want[13:])


@pytest.mark.parametrize("m,d", [(1, 1), (5, 1), (100, 4), (20_000, 800), (4097, 16),
                                 (1 << 20, 2048), (3001, 1_500_000_000)])
def test_countsketch_draws_bit_exact(m, d):
    key = O.derive_seed(11, "countsketch", m)
    rows, signs = _native.rng_countsketch(key, m, d)
    g = O.stream(key)
    want_rows = g.integers(0, d, size=m)
    want_signs = 2.0 * g.integers(0, 2, size=m) - 1.0
    assert np.array_equal(rows, want_rows)
    assert np.array_equal(signs, want_signs)


def test_countsketch_draws_thread_count_invariant():
    key = O.derive_seed(3, "countsketch", 300_001)
    r1, s1 = _native.rng_countsketch(key, 300_001, 800, threads=1)
    r8, s8 = _native.rng_countsketch(key, 300_001, 800, threads=7)
    assert np.array_equal(r1, r8) and np.array_equal(s1, s8)


def test_countsketch_large_digest(golden, golden_meta):
    import hashlib

    m, d, seed = 1 << 22, 8192, 11
    rows, signs = _native.rng_countsketch(O.derive_seed(seed, "countsketch", m), m, d)
    h = hashlib.sha256(rows.tobytes() + signs.tobytes()).hexdigest()
    assert h == golden_meta[f"cs_sha_{m}_{d}_{seed}"]


@pytest.mark.parametrize("m,d,seed", [(50, 16, 2), (1000, 64, 3), (20_000, 800, 4)])
def test_srht_draws_match_golden(golden, golden_meta, m, d, seed):
    m_pad = golden_meta[f"srht_pad_{m}_{d}_{seed}"]
    signs, sample = _native.rng_srht(O.derive_seed(seed, "srht", m), m_pad, d)
    assert np.array_equal(signs, golden[f"srht_signs_{m}_{d}_{seed}"])
    assert np.array_equal(sample, golden[f"srht_sample_{m}_{d}_{seed}"])


@pytest.mark.parametrize("m_pad,d", [(1, 1), (2, 2), (4096, 4096), (1 << 20, 2048)])
def test_srht_draws_match_numpy(m_pad, d):
    key = O.derive_seed(9, "srht", m_pad)
    g = O.stream(key)
    want_signs = (2 * g.integers(0, 2, size=m_pad) - 1).astype(np.int8)
    want_sample = g.permutation(m_pad)[:d]
    signs, sample = _native.rng_srht(key, m_pad, d)
    assert np.array_equal(signs, want_signs)
    assert np.array_equal(sample, want_sample)


@pytest.mark.parametrize("m,d,chunk,warps", [(1, 1, 8, 8), (100, 4, 8, 4), (20_000, 800, 2048, 8),
                                             (65_537, 2048, 2048, 16), (10_000, 8192, 8192, 16),
                                             (9_000, 3, 1024, 8)])
def test_countsketch_plan_structure(m, d, chunk, warps):
    key = O.derive_seed(1, "countsketch", m)
    rows, signs = _native.rng_countsketch(key, m, d)
    ent, tasks, ntask = _native.countsketch_plan(rows, signs, d, chunk, warps)
    stride = int(_native.lib().skl_countsketch_plan_stride(d, warps))
    head = (warps + 1 + 3) // 4 * 4
    nch = (m + chunk - 1) // chunk
    for k in range(nch):
        r0 = k * chunk
        length = min(chunk, m - r0)
        nt = int(ntask[k])
        blk = tasks[k * stride: (k + 1) * stride].astype(np.int64)
        wofs = blk[: warps + 1]
        tk = blk[head: head + nt]
        bkt, start = tk >> 16, tk & 0xFFFF
        ends = np.append(start[1:], length)
        cnts = ends - start
        want_cnt = np.bincount(rows[r0: r0 + length], minlength=d)
        assert nt == np.count_nonzero(want_cnt) and wofs[0] == 0 and wofs[-1] == nt
        assert start[0] == 0 and np.all(cnts >= 1)
        assert np.array_equal(cnts, want_cnt[bkt])          # task = one whole bucket
        for w in range(warps):
            g = slice(wofs[w], wofs[w + 1])
            assert np.all(bkt[g] // -(-d // warps) == w)     # bucket stays in its warp
            assert np.all(np.diff(cnts[g]) <= 0)             # longest first
            ties = np.diff(cnts[g]) == 0
            assert np.all(np.diff(bkt[g])[ties] > 0)         # ties by bucket id
        e = ent[r0: r0 + length].astype(np.int64)
        local, neg = e >> 3, (e & 1).astype(bool)
        assert np.array_equal(np.sort(local), np.arange(length))
        owner = np.repeat(bkt, cnts)
        assert np.array_equal(rows[r0 + local], owner)
        assert np.array_equal(neg, signs[r0 + local] < 0)
        same = owner[1:] == owner[:-1]
        assert np.all(np.diff(local)[same] > 0)             # ascending rows per task


def test_bucket_lists_are_the_csr_of_s():
    m, d = 5000, 37
    rows, signs = _native.rng_countsketch(O.derive_seed(2, "countsketch", m), m, d)
    brow, bptr = _native.countsketch_buckets(rows, d)
    smap = O.countsketch_map(rows.astype(np.int64), signs.astype(np.float64), d, m)
    assert np.array_equal(bptr, smap.indptr)
    assert np.array_equal(brow, smap.indices)


def test_plan_rejects_out_of_range_bucket():
    rows = np.array([0, 5], dtype=np.int32)
    signs = np.array([1, -1], dtype=np.int8)
    with pytest.raises(ValueError):
        _native.countsketch_plan(rows, signs, 4, 8, 8)
    with pytest.raises(Exception):
        _native.countsketch_plan(rows, signs, 70_000, 8, 8)  # d > 65536


def test_gaussian_host_generator_matches_numpy():
    for key in (1, 77, O.derive_seed(3, "gaussian", 262_144)):
        want = O.stream(key).standard_normal(300_000)
        assert np.array_equal(_native.rng_gaussian_host(key, want.size), want)
