"""Oracle pins: conversion, gather, contiguity (CPU only)."""

import random

import numpy as np
import pytest

from oracle import contig, convert, f2
from oracle.constructors import blocked
from oracle.layout import Layout
from workloads import configs
from workloads.values import indices_np, values_np


def L_from_spec(s):
    return Layout(s["in_dims"], s["out_dims"], s["bases"])


def rand_layout(rng, d, dims, zeros=0, out=None):
    """Random distributed layout over a d-bit tensor; ``dims`` = [(name, bits)]
    with sum(bits) = d + zeros (zeros = broadcast columns)."""
    cols = [1 << k for k in range(d)] + [0] * zeros
    rng.shuffle(cols)
    assert sum(b for _, b in dims) == len(cols)
    bases, k = {}, 0
    for n, b in dims:
        bases[n] = [(c,) for c in cols[k:k + b]]
        k += b
    return Layout(dims, out or [("t", d)], bases)


def test_convert_py_equals_np_random():
    rng = random.Random(11)
    for _ in range(60):
        d = rng.randint(2, 9)
        za, zb = rng.randint(0, 2), rng.randint(0, 2)
        na = d + za
        nb = d + zb
        A = rand_layout(rng, d, [("reg", na // 2), ("lane", na - na // 2)], za)
        B = rand_layout(rng, d, [("reg", nb // 3), ("lane", nb - nb // 3)], zb)
        # broadcast-consistent source: src[h] = f(A(h))
        f = values_np(1 << d, 9, 4)
        src = [int(f[f2.apply(A.cols, h)]) for h in range(1 << na)]
        dst = convert.convert_py(src, A, B)
        assert list(convert.convert_np(np.array(src), A, B)) == dst
        # the result is f(B(h)) whatever the tie-break
        assert dst == [int(f[f2.apply(B.cols, h)]) for h in range(1 << nb)]


def test_convert_identity_roundtrip_and_chain():
    rng = random.Random(12)
    for _ in range(40):
        d = rng.randint(2, 10)
        A, B, C = (rand_layout(rng, d, [("reg", 2), ("lane", d - 2)]) for _ in range(3))
        src = list(values_np(1 << d, 1, 2))
        assert convert.convert_py(src, A, A) == src
        mid = convert.convert_py(src, A, B)
        assert convert.convert_py(mid, B, A) == src
        assert convert.convert_py(mid, B, C) == convert.convert_py(src, A, C)


def test_convert_lowest_preimage_tie_break():
    """Broadcast in the source (zero column): the lowest preimage is read
    (reading A4/A6)."""
    A = Layout([("reg", 2)], [("t", 1)], {"reg": [(0,), (1,)]})     # h and h^1 hold the same
    B = Layout([("reg", 1)], [("t", 1)], {"reg": [(1,)]})
    assert convert.convert_py([10, 11, 12, 13], A, B) == [10, 12]


def test_convert_rejects_non_surjective_source():
    A = Layout([("reg", 1)], [("t", 2)], {"reg": [(1,)]})
    B = Layout([("reg", 2)], [("t", 2)], {"reg": [(1,), (2,)]})
    with pytest.raises(ValueError):
        convert.convert_py([1, 2], A, B)


def test_config3_is_numpy_transpose():
    """Special case that reduces to a library routine: row-major ->
    column-major is ndarray.T (SURVEY 8(c) pins)."""
    for m, n in ((4, 4), (5, 3), (3, 6)):
        c = configs.cfg3(n_bits=n, m_bits=m)
        A, B = L_from_spec(c["A"]), L_from_spec(c["B"])
        src = values_np(1 << (m + n), 3, 2)
        dst = convert.convert_np(src, A, B)
        assert (dst == src.reshape(1 << m, 1 << n).T.reshape(-1)).all()


def _cfg2_src_index(b, i, j):
    """mma.sync m16n8 C fragment (PTX ISA: row = groupID + 8*(c>>1), col =
    2*tig + (c&1)), 2 m-tiles x 16 n-tiles per warp, 4 warps along m."""
    g, t = i & 7, (j >> 1) & 3
    lane = g * 4 + t
    e = (j & 1) | (((i >> 3) & 1) << 1)
    reg = e | ((j >> 3) << 2) | (((i >> 4) & 1) << 6)
    warp = (i >> 5) & 3
    return reg | (lane << 7) | (warp << 12) | (b << 14)


def _cfg2_dst_index(b, i, j):
    """Blocked sizePerThread [1,8], threadsPerWarp [2,16], warpsPerCTA [4,1],
    order [1,0] on 128x128, registers repeating along rows."""
    reg = (j & 7) | ((i >> 3) << 3)
    lane = (j >> 3) | ((i & 1) << 4)
    warp = (i >> 1) & 3
    return reg | (lane << 7) | (warp << 12) | (b << 14)


def test_config2_is_ptx_formula_permutation():
    """Config 2 computed without F2: index formulas of the PTX accumulator
    fragment and of the blocked layout."""
    c = configs.cfg2(batch_bits=1)
    A, B = L_from_spec(c["A"]), L_from_spec(c["B"])
    src = values_np(1 << 15, 2, 2)
    dst = convert.convert_np(src, A, B)
    b, i, j = np.meshgrid(np.arange(2), np.arange(128), np.arange(128), indexing="ij")
    si = np.vectorize(_cfg2_src_index)(b, i, j).ravel()
    di = np.vectorize(_cfg2_dst_index)(b, i, j).ravel()
    assert (dst[di] == src[si]).all()


def _cfg6_dst_index(n, k, n_bits, k_bits):
    """Pre-shuffled bf16 operand (reading A25) from the PTX ISA's m16n8k16
    B fragment (.bf16): element b_i of a thread sits at row (k) = 2*tig +
    (i & 1) + 8*(i >> 1), column (n) = groupID, lane = 4*groupID + tig; k-tiles
    k4, k5 are registers 4..15, warps step n by 8, blocks cover (k >> 6) then
    (n >> 5)."""
    kk = k & 15
    i = (kk & 1) | ((kk >> 3) << 1)
    tig = (kk >> 1) & 3
    lane = (n & 7) * 4 + tig
    reg = i | (((k >> 4) & 3) << 2)
    warp = (n >> 3) & 3
    blk = (k >> 6) | ((n >> 5) << (k_bits - 6))
    return reg | (lane << 4) | (warp << 9) | (blk << 11)


def test_config6_preshuffle_is_ptx_fragment_order():
    """Config 6 (the bf16 pre-shuffle) computed without F2: index
    formula of the PTX B fragment."""
    for nb, kb in ((6, 7), (7, 6)):
        c = configs.cfg6(n_bits=nb, k_bits=kb)
        A, B = L_from_spec(c["A"]), L_from_spec(c["B"])
        src = values_np(1 << (nb + kb), 6, 2)
        dst = convert.convert_np(src, A, B)
        n, k = np.meshgrid(np.arange(1 << nb), np.arange(1 << kb), indexing="ij")
        di = np.vectorize(_cfg6_dst_index)(n, k, nb, kb).ravel()
        assert sorted(di.tolist()) == list(range(1 << (nb + kb)))
        assert (dst[di] == src[(n * (1 << kb) + k).ravel()]).all()


def test_convert_np_sampled_equals_full():
    c = configs.cfg5(m_bits=8, kb_bits=7)
    A, B = L_from_spec(c["A"]), L_from_spec(c["B"])
    src = values_np(1 << 15, 6, 1)
    full = convert.convert_np(src, A, B)
    h = np.array([0, 5, 999, 32767, 12345], dtype=np.int64)
    assert (convert.convert_np(src, A, B, h_B=h) == full[h]).all()


def test_gather_is_take_along_axis():
    """tl.gather on a row-major layout equals numpy.take_along_axis."""
    c = configs.cfg4(r_bits=2)
    L = L_from_spec(c["L"])
    n = 1 << L.in_bits
    src = values_np(n, 4, 4)
    idx = indices_np(n, 5, 32)
    out = convert.gather_np(src, idx, L, c["axis"])
    ref = np.take_along_axis(src.reshape(4, 128, 32), idx.reshape(4, 128, 32).astype(np.int64), 2)
    assert (out == ref.reshape(-1)).all()
    # pure python on a slice of it agrees
    small = convert.gather_py(list(src), list(idx), L, c["axis"])
    assert small == list(out)


def test_gather_full_axis_variant():
    c = configs.cfg4(r_bits=1, variant="full")
    L = L_from_spec(c["L"])
    n = 1 << L.in_bits
    src = values_np(n, 4, 4)
    idx = indices_np(n, 5, 4096)
    out = convert.gather_np(src, idx, L, c["axis"])
    ref = np.take_along_axis(src.reshape(2, 4096), idx.reshape(2, 4096).astype(np.int64), 1)
    assert (out == ref.reshape(-1)).all()


def test_gather_rejects_out_of_range():
    c = configs.cfg4(r_bits=0)
    L = L_from_spec(c["L"])
    n = 1 << L.in_bits
    idx = np.zeros(n, dtype=np.int32)
    idx[7] = 32
    with pytest.raises(ValueError):
        convert.gather_np(values_np(n, 1, 4), idx, L, 2)


# ------------------------------------------------------------------ contiguity

def test_contiguity_matrix_A():
    A = blocked([4, 4], R=[1, 1], T=[2, 3], W=[1, 0], order=[1, 0])
    assert contig.contiguous_log2(A) == 1          # reg0 -> j0, reg1 -> i0 breaks the run


@pytest.mark.parametrize("k,w,bits", [
    (1, 2, 64), (2, 2, 128), (4, 2, 128), (8, 2, 128), (16, 2, 128),
    (1, 1, 32), (8, 1, 128), (16, 1, 128)])
def test_contiguity_tab_micro_load_store(k, w, bits):
    """tab:micro-load-store, Triton-Linear bitwidth column, for
    [512, k] tensors loaded by 4 warps with the elements split evenly over the
    128 threads, fastest dim first (partial pin: the paper does not print the
    layouts; the f8 k=2,4 rows need broadcast layouts)."""
    import math
    per_thread = 512 * k // 128
    kb = int(math.log2(k))
    r1 = min(kb, int(math.log2(per_thread)))
    r0 = int(math.log2(per_thread)) - r1
    t1 = kb - r1
    t0 = 5 - t1
    L = blocked([9, kb], R=[r0, r1], T=[t0, t1], W=[9 - r0 - t0, 0], order=[1, 0])
    assert contig.vector_bits(L, w) == bits


# --- chunked whole-buffer evaluation (full-size GPU parity) ------------------------

def test_apply_np_tab_equals_apply_np_and_f2_apply():
    import random
    from oracle import convert as oc
    from oracle import f2 as of2
    rng = random.Random(5)
    for n in (3, 16, 17, 29, 35):
        cols = [rng.getrandbits(40) for _ in range(n)]
        h = np.array([rng.getrandbits(n) for _ in range(2000)], dtype=np.int64)
        a = oc.apply_np_tab(cols, h)
        assert (a == oc.apply_np(cols, h)).all()
        assert all(int(a[i]) == of2.apply(cols, int(h[i])) for i in range(0, 2000, 97))


def test_preimage_table_bij_equals_lowest_preimage_and_rejects_non_bijective():
    from oracle import convert as oc
    from oracle.layout import Layout
    from workloads import configs
    for c in (configs.cfg2(batch_bits=2), configs.cfg3(n_bits=7), configs.cfg5(m_bits=8, kb_bits=7)):
        A = Layout(**c["A"])
        assert (oc.preimage_table_bij_np(A, chunk=1 << 10) == oc.preimage_table_np(A)).all()
    bc = Layout([("reg", 2)], [("i", 2)], {"reg": [(1,), (1,)]})
    with pytest.raises(ValueError):
        oc.preimage_table_bij_np(bc)


def test_convert_np_chunks_concatenate_to_convert_np():
    from oracle import convert as oc
    from oracle.layout import Layout
    from workloads import configs
    from workloads.values import values_np
    for c in (configs.cfg2(batch_bits=2), configs.cfg3(n_bits=7), configs.cfg5(m_bits=8, kb_bits=7)):
        A, B = Layout(**c["A"]), Layout(**c["B"])
        src = values_np(1 << A.in_bits, 3, c["elem_bytes"])
        parts = [d for _, d in oc.convert_np_chunks(src, A, B, chunk=1 << 11)]
        assert np.concatenate(parts).tobytes() == oc.convert_np(src, A, B).tobytes()
