"""The column-threaded C applies of the oracle (oracle/c/apply_oracle.c),
used by the full-size GPU parity tests, against the numpy/scipy
restatement (oracle/oracle.py, itself pinned to the reference's golden
vectors by test_oracle_golden.py): bitwise, including ragged and padded
shapes.  CPU only."""

import numpy as np
import pytest

from oracle import clib
from oracle import oracle as O


@pytest.mark.parametrize("m,n,d", [(1, 1, 1), (7, 3, 2), (1000, 5, 64), (20_000, 9, 800),
                                   (65_537, 2, 2048)])
@pytest.mark.parametrize("threads", [1, 3])
def test_countsketch_fold_mt_bitwise(m, n, d, threads):
    rng = np.random.default_rng(m + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    rows, signs = O.countsketch_draws(O.derive_seed(m, "countsketch", m), m, d)
    want = O.countsketch_apply(rows, signs, d, A)
    got = clib.countsketch_apply_mt(rows, signs, d, A, threads)
    assert np.array_equal(got, want)
    b = rng.standard_normal(m)
    assert np.array_equal(clib.countsketch_apply_mt(rows, signs, d, b, threads),
                          O.countsketch_apply(rows, signs, d, b))


def test_countsketch_fold_mt_column_view():
    rng = np.random.default_rng(2)
    big = np.asfortranarray(rng.standard_normal((3000, 12)))
    view = big[:, 3:8]  # F-contiguous columns, ld = 3000
    rows, signs = O.countsketch_draws(7, 3000, 100)
    assert np.array_equal(clib.countsketch_apply_mt(rows, signs, 100, view),
                          O.countsketch_apply(rows, signs, 100, np.asfortranarray(view)))


@pytest.mark.parametrize("m,n,d", [(1, 1, 1), (5, 2, 3), (4096, 3, 64), (8193, 2, 100),
                                   (20_000, 4, 800), (1 << 15, 2, 2048)])
@pytest.mark.parametrize("threads", [1, 4])
def test_srht_apply_mt_bitwise(m, n, d, threads):
    rng = np.random.default_rng(m * 3 + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    sg, rs, m_pad = O.srht_draws(O.derive_seed(m, "srht", m), m, d)
    want = O.srht_apply(sg, rs, m_pad, d, A)
    got = clib.srht_apply_mt(sg, rs, m_pad, d, A, threads)
    assert np.array_equal(got, want)
    b = rng.standard_normal(m)
    assert np.array_equal(clib.srht_apply_mt(sg, rs, m_pad, d, b, threads),
                          O.srht_apply(sg, rs, m_pad, d, b))
