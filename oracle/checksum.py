"""Buffer checksum (ours, the paper has no such step) --
oracle (tests only).

    indexed:    sum_h fmix(v_h + (base + h + 1) * GAMMA)   mod 2^64
    index-free: sum_h fmix(v_h)                            mod 2^64

v_h = element h as an unsigned integer; fmix = the splitmix64 output function
(Vigna, splitmix64.c).  With v = 0 and base = 0 the indexed terms are the
splitmix64 sequence seeded with 0 (pinned by tests/golden/splitmix64.txt).
"""

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M = (1 << 64) - 1


def fmix(z):
    z &= _M
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


def checksum_py(values, indexed=True, base=0):
    """Plain loop over a sequence of non-negative ints."""
    s = 0
    for h, v in enumerate(values):
        s = (s + fmix(v + (base + h + 1) * GAMMA if indexed else v)) & _M
    return s


def checksum_np(arr, indexed=True, base=0, chunk=1 << 22):
    """The same sum with NumPy uint64 arithmetic (wraps mod 2^64), in chunks."""
    a = np.asarray(arr).reshape(-1)
    a = a.view({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for i in range(0, a.size, chunk):
            v = a[i:i + chunk].astype(np.uint64)
            if indexed:
                h = np.arange(i, i + v.size, dtype=np.uint64) + np.uint64(base + 1)
                z = v + h * np.uint64(GAMMA)
            else:
                z = v
            z = z ^ (z >> np.uint64(30))
            z = z * np.uint64(0xBF58476D1CE4E5B9)
            z = z ^ (z >> np.uint64(27))
            z = z * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            total = total + z.sum(dtype=np.uint64)
    return int(total)
