"""MXFP4 dequantisation -- oracle (tests only).

P:544-549: MXFP4 is "a quantized type where each 32 floating-point elements
share a single 8-bit exponent (i.e., scale)"; the software-emulated
mxfp4 x bf16 path "upcast[s] mxfp4 to bf16".  Element and scale encodings
follow the OCP MX specification the paper cites: E2M1 elements, E8M0
scales 2^(x - 127) with 0xFF = NaN.

upcast_np(packed, A, scales, B) is the plain definition of ll_mxfp4_upcast:
bf16 element 2h + n of the destination holds e2m1(m, 2kb + n) * scale(m, kb),
(m, kb) = B(h), the packed byte read from its lowest preimage under A.
"""

from fractions import Fraction

import numpy as np

from . import convert

# OCP MX E2M1: sign bit 3; exponent bits 2:1 (bias 1); mantissa bit 0
def e2m1_value(code):
    s = -1 if (code >> 3) & 1 else 1
    e = (code >> 1) & 3
    m = code & 1
    mag = Fraction(m, 2) if e == 0 else Fraction(2) ** (e - 1) * (1 + Fraction(m, 2))
    return s, mag


def e8m0_scale(x):
    """2^(x - 127) as a Fraction, or None for NaN (x = 255)."""
    return None if x == 255 else Fraction(2) ** (x - 127)


BF16_MAX = (2 - Fraction(1, 128)) * Fraction(2) ** 127


def bf16_bits(sign, value):
    """bf16 encoding of sign * value for an exactly representable value
    (or one above the range, which becomes inf).  value is a Fraction >= 0."""
    sb = 0x8000 if sign < 0 else 0
    if value == 0:
        return sb
    if value > BF16_MAX:
        return sb | 0x7F80
    f = np.float32(float(value))              # exact: |value| >= 2^-128 and <= 3 significant bits
    if Fraction(float(f)) != value:
        raise ValueError("value not representable")
    bits = int(np.array([f], dtype=np.float32).view(np.uint32)[0])
    if bits & 0xFFFF:
        raise ValueError("value not representable in bf16")
    return sb | (bits >> 16)


def dequant_bits(code, scale_byte):
    """bf16 bits of one element: e2m1(code) * 2^(scale - 127); NaN scale -> NaN."""
    sc = e8m0_scale(scale_byte)
    if sc is None:
        return 0x7FC0
    s, mag = e2m1_value(code)
    return bf16_bits(s, mag * sc)


def dequant_table():
    """[256 scales][16 codes] table of bf16 bits (plain loop over the spec)."""
    return np.array([[dequant_bits(c, x) for c in range(16)] for x in range(256)], dtype=np.uint16)


def upcast_np(packed, A, scales, B, h=None):
    """ll_mxfp4_upcast, whole buffer (or destination byte indices h): returns
    a uint16 array with 2 bf16 per destination byte."""
    kb_bits = B.out_dims[1][1]
    row = 1 << (kb_bits - 4)
    T = convert.preimage_table_np(A)
    if h is None:
        h = np.arange(1 << B.in_bits, dtype=np.int64)
    x = convert.apply_np(B.cols, h)                     # flat (m, kb)
    m = x >> kb_bits
    kb = x & ((1 << kb_bits) - 1)
    byte = np.asarray(packed)[T[x]].astype(np.int64)
    sc = np.asarray(scales)[m * row + (kb >> 4)].astype(np.int64)
    tab = dequant_table()
    out = np.empty(2 * len(h), dtype=np.uint16)
    out[0::2] = tab[sc, byte & 15]
    out[1::2] = tab[sc, byte >> 4]
    return out


def upcast_np_chunks(packed, A, scales, B, chunk=1 << 22):
    """Yields (h0, out[2*h0 : 2*(h0+chunk)]) of ``upcast_np`` over the whole
    destination, chunk by chunk, for a bijective source layout A (the
    evaluation aids of convert.convert_np_chunks; same definition)."""
    kb_bits = B.out_dims[1][1]
    row = 1 << (kb_bits - 4)
    T = convert.preimage_table_bij_np(A)
    tabs = convert._group_tables(B.cols)
    tab = dequant_table()
    packed = np.asarray(packed)
    scales = np.asarray(scales)
    nB = 1 << B.in_bits
    for h0 in range(0, nB, chunk):
        h = np.arange(h0, min(nB, h0 + chunk), dtype=np.int64)
        x = convert.apply_np_tab(B.cols, h, tabs)
        m = x >> kb_bits
        kb = x & ((1 << kb_bits) - 1)
        byte = packed[T[x]].astype(np.int64)
        sc = scales[m * row + (kb >> 4)].astype(np.int64)
        out = np.empty(2 * len(h), dtype=np.uint16)
        out[0::2] = tab[sc, byte & 15]
        out[1::2] = tab[sc, byte >> 4]
        yield h0, out
