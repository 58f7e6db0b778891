"""The BASELINE.json workloads as literal layout tables.

A layout spec is a dict ``{"in_dims": [(name, bits)...], "out_dims": [(name,
bits)...], "bases": {name: [coords per out dim, ...]}}`` -- exactly the
arguments of the C-ABI ``ll_layout_create`` (include/ll.h) and of
``oracle.layout.Layout``.  Bits are written by name ("j3" = bit 3 of tensor
dim j) to keep the tables readable; ``_b`` only turns a name into a
one-hot coordinate tuple.  Sizes are parameters so that tests can run the same
layout family at oracle-friendly sizes; the defaults are the benchmark sizes.
"""


def _b(out_dims, name):
    """One-hot coordinate tuple for bit ``name`` = '<dim><k>' (or 0 for zero)."""
    if name == "0":
        return tuple(0 for _ in out_dims)
    for d, (dn, _) in enumerate(out_dims):
        if name.startswith(dn) and name[len(dn):].isdigit():
            k = int(name[len(dn):])
            return tuple((1 << k) if e == d else 0 for e in range(len(out_dims)))
    raise KeyError(name)


def spec(in_names_bits, out_dims):
    """in_names_bits: list of (in_dim, [bit names]) -> layout spec dict."""
    return {
        "in_dims": [(n, len(bits)) for n, bits in in_names_bits],
        "out_dims": list(out_dims),
        "bases": {n: [_b(out_dims, x) for x in bits] for n, bits in in_names_bits},
    }


def _rng(prefix, lo, hi):
    return ["%s%d" % (prefix, k) for k in range(lo, hi)]


# --- config 1: paper Fig. 1, 16x16 fp16, 2 warps -------------------------------------

def cfg1(variant="mma"):
    """A = matrix A of P:283-295; B = reading A3 (1a: mma C fragment over two
    warps along j; 1b: A with i and j exchanged)."""
    out = [("i", 4), ("j", 4)]
    A = spec([("reg", ["j0", "i0"]), ("lane", ["j1", "j2", "j3", "i1", "i2"]),
              ("warp", ["i3"])], out)
    if variant == "mma":
        B = spec([("reg", ["j0", "i3"]), ("lane", ["j1", "j2", "i0", "i1", "i2"]),
                  ("warp", ["j3"])], out)
    elif variant == "T":
        B = spec([("reg", ["i0", "j0"]), ("lane", ["i1", "i2", "i3", "j1", "j2"]),
                  ("warp", ["j3"])], out)
    else:
        raise ValueError(variant)
    return dict(name="cfg1" + ("a" if variant == "mma" else "b"), A=A, B=B, elem_bytes=2)


# --- config 2: mma.sync m16n8k16 accumulator -> blocked, 128x128 fp16 tiles ----------

def cfg2(batch_bits=12):
    out = [("b", batch_bits), ("i", 7), ("j", 7)]
    blk = ("block", _rng("b", 0, batch_bits))
    A = spec([("reg", ["j0", "i3", "j3", "j4", "j5", "j6", "i4"]),
              ("lane", ["j1", "j2", "i0", "i1", "i2"]), ("warp", ["i5", "i6"]), blk], out)
    B = spec([("reg", ["j0", "j1", "j2", "i3", "i4", "i5", "i6"]),
              ("lane", ["j3", "j4", "j5", "j6", "i0"]), ("warp", ["i1", "i2"]), blk], out)
    return dict(name="cfg2", A=A, B=B, elem_bytes=2)


def cfg2w(batch_bits=12):
    """SURVEY 8(a) a5, "cfg2 warp-aligned variant": the mma C fragment ->
    a blocked-style layout that keeps the warps on [i5, i6] (8 fp16 per
    thread along j, 16 x 2 threads, the remaining rows as register
    repetitions), so (B^-1 o A)_warp = I and the paper's warp-shuffle
    exchange applies; 64 rounds."""
    out = [("b", batch_bits), ("i", 7), ("j", 7)]
    blk = ("block", _rng("b", 0, batch_bits))
    A = spec([("reg", ["j0", "i3", "j3", "j4", "j5", "j6", "i4"]),
              ("lane", ["j1", "j2", "i0", "i1", "i2"]), ("warp", ["i5", "i6"]), blk], out)
    B = spec([("reg", ["j0", "j1", "j2", "i1", "i2", "i3", "i4"]),
              ("lane", ["j3", "j4", "j5", "j6", "i0"]), ("warp", ["i5", "i6"]), blk], out)
    return dict(name="cfg2w", A=A, B=B, elem_bytes=2)


# --- config 3: row-major -> column-major transpose, 2^n x 2^n bf16 -----------------

def cfg3(n_bits=13, m_bits=None):
    m_bits = n_bits if m_bits is None else m_bits
    out = [("i", m_bits), ("j", n_bits)]
    A = spec([("offset", _rng("j", 0, n_bits) + _rng("i", 0, m_bits))], out)
    B = spec([("offset", _rng("i", 0, m_bits) + _rng("j", 0, n_bits))], out)
    return dict(name="cfg3", A=A, B=B, elem_bytes=2)


# --- config 4: warp-shuffle gather, fp32 + int32 indices -----------------------------

def cfg4(r_bits=12, variant="tile"):
    """Reading A21: tile-local gather on the [2^r, 128, 32] view, axis = last
    (primary), or the full 4096-long axis of a [2^r, 4096] view (variant)."""
    if variant == "tile":
        out = [("r", r_bits), ("s", 7), ("k", 5)]
        L = spec([("reg", ["k0", "k1"]), ("lane", ["k2", "k3", "k4", "s0", "s1"]),
                  ("warp", ["s2", "s3"]), ("block", ["s4", "s5", "s6"] + _rng("r", 0, r_bits))], out)
        return dict(name="cfg4", L=L, axis=2, elem_bytes=4, idx_limit=32)
    out = [("r", r_bits), ("c", 12)]
    L = spec([("reg", ["c0", "c1"]), ("lane", _rng("c", 2, 7)), ("warp", ["c7", "c8"]),
              ("block", ["c9", "c10", "c11"] + _rng("r", 0, r_bits))], out)
    return dict(name="cfg4full", L=L, axis=1, elem_bytes=4, idx_limit=4096)


# --- config 5: mxfp4 packed-byte layout conversion ------------------------------------

def cfg5(m_bits=15, kb_bits=14):
    """Reading A22: A = coalesced blocked bytes (16 B per thread along K);
    B = packed image of the bf16 m16n8k16 A fragment.  Tile = 128 rows x 64 B."""
    out = [("m", m_bits), ("kb", kb_bits)]
    blk = ("block", _rng("kb", 6, kb_bits) + _rng("m", 7, m_bits))
    A = spec([("reg", ["kb0", "kb1", "kb2", "kb3", "m5", "m6"]),
              ("lane", ["kb4", "kb5", "m0", "m1", "m2"]), ("warp", ["m3", "m4"]), blk], out)
    B = spec([("reg", ["m3", "kb2", "kb3", "kb4", "kb5", "m6"]),
              ("lane", ["kb0", "kb1", "m0", "m1", "m2"]), ("warp", ["m4", "m5"]), blk], out)
    return dict(name="cfg5", A=A, B=B, elem_bytes=1)


# --- pre-shuffle: bf16 operand -> fragment order ------

def cfg6(n_bits=13, k_bits=13):
    """Reading A25: the HBM pre-shuffle of a bf16 [N, K] operand.
    A = row-major memory layout (k fastest).  B = the bf16 mma m16n8k16
    B-operand fragment (reg [k0, k3], lane [k1, k2, n0, n1, n2], reading A8)
    with two more k-tiles as register bits (k4, k5: 8 bf16 = 16 B per thread,
    so a consumer loads its fragments with one 128-bit load), 4 warps along n
    (n3, n4), blocks over the rest -- the destination buffer in
    hardware-index order."""
    out = [("n", n_bits), ("k", k_bits)]
    B = spec([("reg", ["k0", "k3", "k4", "k5"]), ("lane", ["k1", "k2", "n0", "n1", "n2"]),
              ("warp", ["n3", "n4"]), ("block", _rng("k", 6, k_bits) + _rng("n", 5, n_bits))], out)
    A = spec([("offset", _rng("k", 0, k_bits) + _rng("n", 0, n_bits))], out)
    return dict(name="cfg6", A=A, B=B, elem_bytes=2)


def total_elems(spec_):
    return 1 << sum(b for _, b in spec_["in_dims"])
