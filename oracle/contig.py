"""Contiguity / vector width -- oracle (tests only).

"Contiguous elements": the number of contiguous elements per
thread is the largest contiguous block of the logical tensor that the inverse
of the layout maps identically onto registers: the largest u with
L^{-1}_reg(i) = i for all i <= u.
"""

from . import f2


def contiguous_log2(L):
    """Largest k such that tensor flat bits 0..k-1 are mapped by L^{-1} onto
    register bits 0..k-1 identically."""
    inv = f2.right_inverse(L.cols, L.out_bits)      # tensor flat bit -> hardware flat index
    roff = L.in_offset("reg")
    nreg = L.in_size("reg")
    k = 0
    while k < L.out_bits and k < nreg and inv[k] == 1 << (roff + k):
        k += 1
    return k


def vector_bits(L, elem_bytes, max_bits=128):
    """Width in bits of one vectorised global access: 2^k elements, capped at
    the 128-bit vector instruction (tab:micro-load-store)."""
    return min(max_bits, (1 << contiguous_log2(L)) * elem_bytes * 8)
