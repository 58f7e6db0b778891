"""Counter-based seeded values (splitmix64) -- NumPy and PyTorch versions.

value(h, seed) = splitmix64(h + seed * 2^40), truncated to the element width.
Every element of a test buffer is a distinct pseudo-random pattern of its
index, so any misplaced element is visible in a byte-exact comparison.
Both implementations compute the same integers (tested).
"""

import numpy as np

_G = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_DT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


def splitmix64_np(x):
    z = np.asarray(x, dtype=np.uint64) + np.uint64(_G)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def values_np(n, seed, elem_bytes, start=0):
    """n values for indices start..start+n-1 as a uint array of the width."""
    with np.errstate(over="ignore"):
        h = np.arange(start, start + n, dtype=np.uint64) + np.uint64(seed << 40)
        return splitmix64_np(h).astype(_DT[elem_bytes])


def indices_np(n, seed, limit, start=0):
    """Gather indices uniform in [0, limit) (limit a power of two), int32."""
    with np.errstate(over="ignore"):
        h = np.arange(start, start + n, dtype=np.uint64) + np.uint64(seed << 40)
        return (splitmix64_np(h) & np.uint64(limit - 1)).astype(np.int32)


def _lsr(z, k):
    import torch
    return (z >> k) & torch.tensor((1 << (64 - k)) - 1, dtype=torch.int64, device=z.device)


def _s64(c):
    return c - (1 << 64) if c >= (1 << 63) else c


def splitmix64_torch(h):
    """Same as splitmix64_np on an int64 tensor (two's-complement wrap)."""
    z = h + _s64(_G)
    z = (z ^ _lsr(z, 30)) * _s64(_M1)
    z = (z ^ _lsr(z, 27)) * _s64(_M2)
    return z ^ _lsr(z, 31)


_TDT = {1: "uint8", 2: "int16", 4: "int32", 8: "int64"}


def values_torch(n, seed, elem_bytes, device, start=0, chunk=1 << 26):
    """Device-side generation of ``values_np``; returns a uint8/int16/int32/int64
    tensor (raw bits; compare as bytes)."""
    import torch
    out = torch.empty(n, dtype=getattr(torch, _TDT[elem_bytes]), device=device)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        h = torch.arange(start + c0, start + c1, dtype=torch.int64, device=device) + (seed << 40)
        z = splitmix64_torch(h)
        if elem_bytes == 8:
            out[c0:c1] = z
        else:
            z = z & ((1 << (8 * elem_bytes)) - 1)
            if elem_bytes == 1:
                out[c0:c1] = z.to(torch.uint8)
            else:   # reinterpret the low bits as signed of the same width
                half = 1 << (8 * elem_bytes - 1)
                out[c0:c1] = torch.where(z >= half, z - 2 * half, z).to(out.dtype)
    return out


def indices_torch(n, seed, limit, device, start=0):
    import torch
    h = torch.arange(start, start + n, dtype=torch.int64, device=device) + (seed << 40)
    return (splitmix64_torch(h) & (limit - 1)).to(torch.int32)
