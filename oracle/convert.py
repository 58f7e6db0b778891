"""Layout conversion and gather: the plain definitions -- oracle (tests only).

``convert`` is the conversion B^{-1} o A of P:599-611 read as a *pull*
(reading A6): every destination slot h_B receives the value held by the
lowest source index h_A with A(h_A) = B(h_B).  ``gather`` is ``tl.gather``
(P:719-722): out(x) = src(x with its ``axis`` coordinate replaced by idx(x)).

Buffer convention: a buffer for layout L holds 2^{in_bits(L)}
elements; the element at flattened input index h holds tensor element L(h).

``*_py`` are pure-Python element loops (small cases); ``*_np`` compute the
same definition with NumPy over whole buffers (P:, no reordering: build the
table, then index), used where pure Python would take minutes.
"""

import numpy as np

from . import f2


# --- pure Python ----------------------------------------------------------------

def preimage_table_py(A):
    """T[x] = min{h : A(h) = x}; None where x has no preimage."""
    cols = A.cols
    T = [None] * (1 << A.out_bits)
    for h in range(1 << A.in_bits):
        x = f2.apply(cols, h)
        if T[x] is None:
            T[x] = h
    return T


def convert_py(src, A, B):
    """dst[h_B] = src[T[B(h_B)]] (reading A6).  Raises if some B(h_B) is
    not in the image of A."""
    if [n for n in A.out_dims] != [n for n in B.out_dims]:
        raise ValueError("convert: layouts map to different tensors")
    if len(src) != (1 << A.in_bits):
        raise ValueError("convert: src has the wrong size")
    T = preimage_table_py(A)
    bcols = B.cols
    dst = []
    for h in range(1 << B.in_bits):
        x = f2.apply(bcols, h)
        if T[x] is None:
            raise ValueError("convert: tensor element %d is not held by the source layout" % x)
        dst.append(src[T[x]])
    return dst


def axis_field(L, axis):
    """(shift, nbits) of output dim ``axis`` in the flat tensor index."""
    return L.out_shift(axis), L.out_dims[axis][1]


def gather_py(src, idx, L, axis):
    """``tl.gather``: out[h] = src[T[L(h) with axis <- idx[h]]]."""
    T = preimage_table_py(L)
    shift, nb = axis_field(L, axis)
    mask = ((1 << nb) - 1) << shift
    cols = L.cols
    out = []
    for h in range(1 << L.in_bits):
        i = int(idx[h])
        if i < 0 or i >= (1 << nb):
            raise ValueError("gather: index %d out of range" % i)
        y = (f2.apply(cols, h) & ~mask) | (i << shift)
        out.append(src[T[y]])
    return out


# --- NumPy (whole buffers) ----------------------------------------------------------

def apply_np(cols, h):
    """Vectorised f2.apply: XOR of the columns selected by the bits of h."""
    h = np.asarray(h, dtype=np.int64)
    out = np.zeros_like(h)
    for k, c in enumerate(cols):
        if c:
            out ^= np.where((h >> k) & 1, np.int64(c), np.int64(0))
    return out


def preimage_table_np(A):
    """T[x] = min{h : A(h) = x}, or -1."""
    n = A.in_bits
    h = np.arange(1 << n, dtype=np.int64)
    x = apply_np(A.cols, h)
    T = np.full(1 << A.out_bits, -1, dtype=np.int64)
    order = np.argsort(x, kind="stable")          # stable: equal x keep h ascending
    xs = x[order]
    first = np.ones(len(xs), dtype=bool)
    first[1:] = xs[1:] != xs[:-1]
    T[xs[first]] = order[first]
    return T


def convert_np(src, A, B, h_B=None):
    """NumPy version of ``convert_py``.  If ``h_B`` is given, only those
    destination indices are computed (sampled parity at full size)."""
    src = np.asarray(src)
    if src.shape[0] != (1 << A.in_bits):
        raise ValueError("convert: src has the wrong size")
    T = preimage_table_np(A)
    if h_B is None:
        h_B = np.arange(1 << B.in_bits, dtype=np.int64)
    x = apply_np(B.cols, h_B)
    t = T[x]
    if (t < 0).any():
        raise ValueError("convert: some tensor element is not held by the source layout")
    return src[t]


def gather_np(src, idx, L, axis, h=None):
    src = np.asarray(src)
    idx = np.asarray(idx).astype(np.int64)
    T = preimage_table_np(L)
    shift, nb = axis_field(L, axis)
    mask = ((1 << nb) - 1) << shift
    if h is None:
        h = np.arange(1 << L.in_bits, dtype=np.int64)
        ih = idx
    else:
        ih = idx[h]
    if (ih < 0).any() or (ih >= (1 << nb)).any():
        raise ValueError("gather: index out of range")
    y = (apply_np(L.cols, h) & ~np.int64(mask)) | (ih << shift)
    return src[T[y]]


# --- whole buffers at full size (chunked) --------------------------------------------
#
# The same definitions, evaluated over 2^26-2^29-element buffers in chunks
# (GPU parity on the BASELINE sizes).  Two evaluation aids, both pinned
# against the functions above in tests/test_oracle_convert.py:
#   * apply_np_tab: the location of an index is the XOR of the locations of
#     its parts ("the XOR of per-level locations"); the input bits are
#     cut into groups of <= 16 bits, each group's 2^16 XOR-combinations are
#     tabulated with apply_np, and a point is the XOR of its groups' entries;
#   * preimage_table_bij_np: for a bijective layout the lowest preimage is the
#     only preimage, so T is the inverse permutation, T[A(h)] = h (no sort).

def _group_tables(cols, group_bits=16):
    tabs = []
    for g0 in range(0, len(cols), group_bits):
        part = cols[g0:g0 + group_bits]
        tabs.append((g0, len(part), apply_np(part, np.arange(1 << len(part), dtype=np.int64))))
    return tabs


def apply_np_tab(cols, h, tabs=None):
    """apply_np(cols, h) as the XOR of per-group table entries."""
    h = np.asarray(h, dtype=np.int64)
    if tabs is None:
        tabs = _group_tables(cols)
    out = np.zeros_like(h)
    for g0, nb, tab in tabs:
        out ^= tab[(h >> g0) & ((1 << nb) - 1)]
    return out


def preimage_table_bij_np(A, chunk=1 << 22):
    """T[x] = the preimage of x under a bijective A (in_bits == out_bits and
    every x hit exactly once; ValueError otherwise)."""
    n = A.in_bits
    if n != A.out_bits:
        raise ValueError("preimage_table_bij_np: layout is not square")
    T = np.full(1 << n, -1, dtype=np.int64)
    tabs = _group_tables(A.cols)
    for h0 in range(0, 1 << n, chunk):
        h = np.arange(h0, min(1 << n, h0 + chunk), dtype=np.int64)
        T[apply_np_tab(A.cols, h, tabs)] = h
    if (T < 0).any():
        raise ValueError("preimage_table_bij_np: layout is not bijective")
    return T


def convert_np_chunks(src, A, B, chunk=1 << 22):
    """Yields (h0, dst[h0:h0+chunk]) of ``convert_np(src, A, B)`` for a
    bijective source layout A: dst[h_B] = src[T[B(h_B)]] chunk by chunk."""
    src = np.asarray(src)
    if src.shape[0] != (1 << A.in_bits):
        raise ValueError("convert: src has the wrong size")
    T = preimage_table_bij_np(A)
    tabs = _group_tables(B.cols)
    nB = 1 << B.in_bits
    for h0 in range(0, nB, chunk):
        h = np.arange(h0, min(nB, h0 + chunk), dtype=np.int64)
        yield h0, src[T[apply_np_tab(B.cols, h, tabs)]]
