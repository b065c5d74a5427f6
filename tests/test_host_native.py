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


def _simulate_plan(lanes, off, d, chunk, warps, m, A):
    """Execute the lane lists exactly as countsketch_dense_kernel does
    (per warp: 32 lanes holding (bucket, running sum), write back / reload on
    a bucket change, stores before loads within a step)."""
    head = (warps + 1 + 3) // 4 * 4
    acc = np.zeros(d + 1)
    cur = np.full((warps, 32), d)
    a = np.zeros((warps, 32))
    for k in range(len(off) - 1):
        blk = lanes[off[k]: off[k + 1]].astype(np.int64)
        wrow = blk[: warps + 1]
        words = blk[head:].reshape(-1, 32)
        r0 = k * chunk
        stage = np.zeros(chunk + 1)
        seg = A[r0: r0 + chunk]
        stage[: len(seg)] = seg
        for w in range(warps):
            for row in words[wrow[w]: wrow[w + 1]]:
                j = (row & 0x7FFF) // 8
                x = stage[j] * np.where(row >> 31, -1.0, 1.0)
                b = (row >> 16) & 0x7FFF
                sw = b != cur[w]
                acc[cur[w][sw]] = a[w][sw]          # write back (distinct buckets)
                cur[w][sw] = b[sw]
                a[w][sw] = acc[b[sw]]
                a[w] = a[w] + x
    for w in range(warps):
        for l in range(32):
            acc[cur[w][l]] = a[w][l]
    return acc[:d]


@pytest.mark.parametrize("m,d,chunk,warps", [(1, 1, 8, 8), (100, 4, 8, 4), (20_000, 800, 2048, 8),
                                             (65_537, 2048, 2048, 16), (10_000, 8192, 4088, 16),
                                             (9_000, 3, 1024, 8), (200_000, 2048, 2048, 16)])
def test_countsketch_plan_structure_and_semantics(m, d, chunk, warps):
    key = O.derive_seed(1, "countsketch", m)
    rows, signs = _native.rng_countsketch(key, m, d)
    lanes, off, mx = _native.countsketch_plan(rows, signs, d, chunk, warps)
    head = (warps + 1 + 3) // 4 * 4
    gsize = -(-d // warps)
    nch = (m + chunk - 1) // chunk
    assert off[0] == 0 and len(off) == nch + 1 and mx == int(np.diff(off).max())
    for k in range(0, nch, max(1, nch // 7)):
        r0 = k * chunk
        length = min(chunk, m - r0)
        blk = lanes[off[k]: off[k + 1]].astype(np.int64)
        wrow = blk[: warps + 1]
        words = blk[head:]
        assert len(words) == 32 * wrow[warps] and wrow[0] == 0 and np.all(np.diff(wrow) >= 0)
        seen = np.zeros(length, dtype=int)
        for w in range(warps):
            sub = words[32 * wrow[w]: 32 * wrow[w + 1]].reshape(-1, 32)
            owner = {}
            for lane in range(32):
                lst = sub[:, lane]
                real = (lst & 0x7FFF) != 8 * chunk
                j = (lst[real] & 0x7FFF) // 8
                bkt = (lst[real] >> 16) & 0x7FFF
                neg = (lst[real] >> 31) & 1
                seen[j] += 1
                assert np.all(rows[r0 + j] == bkt)            # entry -> its bucket
                assert np.all(bkt // gsize == w)              # bucket stays in its warp
                assert np.array_equal(neg.astype(bool), signs[r0 + j] < 0)
                for b in np.unique(bkt):
                    pos = np.flatnonzero(bkt == b)
                    assert np.all(np.diff(pos) == 1)          # one contiguous run ...
                    assert np.all(np.diff(j[pos]) > 0)        # ... in ascending rows
                    assert owner.setdefault(int(b), lane) == lane
                pads = (lst[~real] >> 16) & 0x7FFF
                assert np.all(pads <= d)
        assert np.all(seen == 1)                              # every row exactly once
    # executing the lists reproduces the reference fold bitwise
    if m <= 200_000:
        A = np.random.default_rng(m).standard_normal(m)
        got = _simulate_plan(lanes, off, d, chunk, warps, m, A)
        want = O.countsketch_fold(rows.astype(np.int64), signs.astype(np.float64), d, A)
        assert np.array_equal(got, want)


def _simulate_owned(lanes, off, d, chunk, warps, m, x):
    """Execute a register-owned plan the way the kernel does: every lane
    folds its list in order into the register of the entry's slot."""
    head = (warps + 1 + 7) // 8 * 8
    acc = np.zeros((warps, 32, 4))
    for k in range(len(off) - 1):
        r0 = k * chunk
        xs = np.zeros(chunk + 1)
        seg = x[r0: r0 + chunk]
        xs[: len(seg)] = seg
        blk = lanes[off[k]: off[k + 1]].astype(np.int64)
        for w in range(warps):
            sub = blk[head + 32 * blk[w]: head + 32 * blk[w + 1]].reshape(-1, 32)
            for step in sub:
                v = np.where(step >> 15, -1.0, 1.0) * xs[step & 0x1FFF]
                acc[w, np.arange(32), (step >> 13) & 3] += v
    # slot q of thread t owns bucket t + q * 32 * warps
    return acc.reshape(32 * warps, 4).T.reshape(-1)[:d]


@pytest.mark.parametrize("m,d,chunk,warps", [(1, 1, 8, 8), (100, 4, 8, 8), (20_000, 800, 8184, 8),
                                             (65_537, 2048, 8184, 16), (9_000, 3, 1024, 8),
                                             (50_000, 1024, 4096, 8), (30_001, 1025, 8184, 16)])
def test_owned_plan_structure_and_semantics(m, d, chunk, warps):
    """Register-owned plan (skl_countsketch_plan_owned): every row exactly
    once, in the lane/slot that owns its bucket, ascending within a bucket,
    and executing it reproduces the scipy fold bitwise."""
    key = O.derive_seed(5, "countsketch", m)
    rows, signs = _native.rng_countsketch(key, m, d)
    lanes, off, mx = _native.countsketch_plan_owned(rows, signs, d, chunk, warps)
    head = (warps + 1 + 7) // 8 * 8
    nch = (m + chunk - 1) // chunk
    assert lanes.dtype == np.uint16 and off[0] == 0 and len(off) == nch + 1
    assert mx == int(np.diff(off).max()) and np.all(np.diff(off) % 8 == 0)
    for k in range(0, nch, max(1, nch // 5)):
        r0 = k * chunk
        length = min(chunk, m - r0)
        blk = lanes[off[k]: off[k + 1]].astype(np.int64)
        wrow = blk[: warps + 1]
        assert wrow[0] == 0 and np.all(np.diff(wrow) >= 0)
        assert len(blk) == head + 32 * wrow[warps]
        seen = np.zeros(length, dtype=int)
        for w in range(warps):
            sub = blk[head + 32 * wrow[w]: head + 32 * wrow[w + 1]].reshape(-1, 32)
            for lane in range(32):
                lst = sub[:, lane]
                j = lst & 0x1FFF
                real = j != chunk
                jr, slot = j[real], (lst[real] >> 13) & 3
                assert np.all((lst[~real] >> 13) == 0)          # pads: slot 0, +, zero row
                seen[jr] += 1
                assert np.all(rows[r0 + jr] == w * 32 + lane + slot * 32 * warps)
                assert np.array_equal(((lst[real] >> 15) & 1).astype(bool), signs[r0 + jr] < 0)
                for s_ in range(4):
                    assert np.all(np.diff(jr[slot == s_]) > 0)  # ascending per bucket
        assert np.all(seen == 1)
    x = np.random.default_rng(m).standard_normal(m)
    got = _simulate_owned(lanes, off, d, chunk, warps, m, x)
    want = O.countsketch_fold(rows.astype(np.int64), signs.astype(np.float64), d, x)
    assert np.array_equal(got, want)


def test_owned_plan_limits_and_thread_invariance():
    m, d = 100_000, 2048
    rows, signs = _native.rng_countsketch(O.derive_seed(6, "countsketch", m), m, d)
    l1, o1, _ = _native.countsketch_plan_owned(rows, signs, d, 8184, 16, threads=1)
    l7, o7, _ = _native.countsketch_plan_owned(rows, signs, d, 8184, 16, threads=7)
    assert np.array_equal(o1, o7) and np.array_equal(l1, l7)
    with pytest.raises(Exception):
        _native.countsketch_plan_owned(rows, signs, d, 8184, 8)     # 2048 > 8 warps x 128
    with pytest.raises(Exception):
        _native.countsketch_plan_owned(rows, signs, d, 8192, 16)    # row field is 13 bits
    bad = rows.copy()
    bad[7] = d
    with pytest.raises(ValueError):
        _native.countsketch_plan_owned(bad, signs, d, 8184, 16)


def test_plan_is_thread_count_invariant():
    m, d = 300_000, 2048
    rows, signs = _native.rng_countsketch(O.derive_seed(4, "countsketch", m), m, d)
    l1, o1, _ = _native.countsketch_plan(rows, signs, d, 2048, 16, threads=1)
    l8, o8, _ = _native.countsketch_plan(rows, signs, d, 2048, 16, threads=7)
    assert np.array_equal(o1, o8) and np.array_equal(l1, l8)


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
        _native.countsketch_plan(rows, signs, 40_000, 8, 8)  # d > 32767


def test_gaussian_host_generator_matches_numpy():
    for key in (1, 77, O.derive_seed(3, "gaussian", 262_144)):
        want = O.stream(key).standard_normal(300_000)
        assert np.array_equal(_native.rng_gaussian_host(key, want.size), want)
