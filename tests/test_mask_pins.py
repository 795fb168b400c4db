"""Pins of the RM/FM mask oracle (oracle/masks.py), -m "not gpu".

The key stream is pinned to splitmix64's published reference outputs (state 0), the k-smallest
selection to a brute-force sort in Python integers on tiny inputs, and the protocols to their
defining properties (exact counts, nesting in k, whole fibres, uniform inclusion)."""
import itertools

import numpy as np
import pytest

from oracle import masks as MK


def test_splitmix64_reference_outputs():
    # splitmix64 (Steele, Lea, Flood 2014; Vigna's reference C) from state 0: its first three
    # outputs are the widely quoted test vectors below.
    k = MK.splitmix64_keys(0, 3)
    assert [int(v) for v in k] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_keys_distinct_and_seeded():
    a = MK.splitmix64_keys(7, 100000)
    assert np.unique(a).size == a.size
    b = MK.splitmix64_keys(8, 100000)
    assert not np.array_equal(a, b)
    # the stream from seed s shifted by one step equals the stream from s + gamma
    c = MK.splitmix64_keys((7 + 0x9E3779B97F4A7C15) % 2**64, 99999)
    assert np.array_equal(a[1:], c)
    assert np.array_equal(MK.splitmix64_keys(7, 500, start=99500), a[99500:])


@pytest.mark.parametrize("n,k", [(1, 0), (1, 1), (7, 3), (33, 10), (64, 64), (50, 1)])
def test_uniform_matches_brute_force(n, k):
    seed = 12345
    keys = [int(v) for v in MK.splitmix64_keys(seed, n)]
    want = set(sorted(range(n), key=lambda u: keys[u])[:k])
    got = MK.mask_uniform(n, k, seed)
    assert got.dtype == np.uint8 and got.size == n
    assert set(np.flatnonzero(got).tolist()) == want


def test_uniform_exact_count_and_nesting():
    n = 10007
    prev = MK.mask_uniform(n, 0, 3)
    assert prev.sum() == 0
    for k in (1, 500, 1001, 5000, 10006, 10007):
        m = MK.mask_uniform(n, k, 3)
        assert int(m.sum()) == k
        assert np.all(m >= prev)          # k smallest ⊂ k' smallest for k < k'
        prev = m


def test_uniform_inclusion_is_uniform():
    # every index is included with probability k/n; over S seeds the count per index is
    # Binomial(S, k/n): check the chi-square statistic against its mean n-1 (sd √(2(n−1))).
    n, k, S = 200, 50, 400
    cnt = np.zeros(n)
    for s in range(S):
        cnt += MK.mask_uniform(n, k, s)
    p = k / n
    chi2 = np.sum((cnt - S * p) ** 2 / (S * p * (1 - p)))
    assert abs(chi2 - (n - 1)) < 6 * np.sqrt(2 * (n - 1))


@pytest.mark.parametrize("dims,mode,missing", [((4, 3, 5), 0, 6), ((4, 3, 5), 1, 11), ((4, 3, 5), 2, 0),
                                               ((2, 3, 4, 5), 2, 29), ((2, 3, 4, 5), 3, 24), ((6,), 0, 1)])
def test_fibres_brute_force(dims, mode, missing):
    seed = 99
    got = MK.mask_fibres(dims, mode, missing, seed)
    other = [d for m, d in enumerate(dims) if m != mode]
    nf = int(np.prod(other)) if other else 1
    keys = [int(v) for v in MK.splitmix64_keys(seed, nf)]
    miss = set(sorted(range(nf), key=lambda f: keys[f])[:missing])
    # explicit multi-index walk: linear index (mode-1 fastest) and fibre id (mode removed)
    for idx in itertools.product(*[range(d) for d in dims]):
        u, mul = 0, 1
        for m, d in enumerate(dims):
            u += idx[m] * mul
            mul *= d
        f, mul = 0, 1
        for m, d in enumerate(dims):
            if m != mode:
                f += idx[m] * mul
                mul *= d
        assert got[u] == (0 if f in miss else 1)
    assert int((got == 0).sum()) == missing * dims[mode]
