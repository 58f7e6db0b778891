"""Oracle checksum (row a12) against the splitmix64 reference outputs and the
sum's algebraic properties (CPU only)."""

import os

import numpy as np

from oracle import checksum as ck

GOLD = os.path.join(os.path.dirname(__file__), "golden", "splitmix64.txt")


def _golden():
    return [int(l, 16) for l in open(GOLD) if l.strip() and not l.startswith("#")]


def test_zero_buffer_is_splitmix64_sequence():
    g = _golden()
    for k in range(1, len(g) + 1):
        assert ck.checksum_py([0] * k) == sum(g[:k]) % (1 << 64)
        assert ck.checksum_np(np.zeros(k, dtype=np.uint32)) == sum(g[:k]) % (1 << 64)


def test_partition_additivity_and_np_equals_py():
    rng = np.random.default_rng(3)
    for dt in (np.uint8, np.uint16, np.uint32, np.uint64):
        a = rng.integers(0, np.iinfo(dt).max, 1001, dtype=dt, endpoint=True)
        whole = ck.checksum_py([int(x) for x in a])
        assert ck.checksum_np(a, chunk=97) == whole
        for cut in (0, 1, 500, 1001):
            s = (ck.checksum_np(a[:cut]) + ck.checksum_np(a[cut:], base=cut)) % (1 << 64)
            assert s == whole


def test_index_free_sum_is_permutation_invariant_indexed_is_not():
    rng = np.random.default_rng(4)
    a = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)
    p = rng.permutation(a)
    assert ck.checksum_np(a, indexed=False) == ck.checksum_np(p, indexed=False)
    b = a.copy()
    i, j = 10, 20
    assert b[i] != b[j]
    b[i], b[j] = b[j], b[i]
    assert ck.checksum_np(a) != ck.checksum_np(b)
