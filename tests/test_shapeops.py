"""Shape-operation transfer functions, CPU only.

* the C ABI (ll_transpose / ll_reshape / ll_expand_dims / ll_broadcast /
  ll_join / ll_split) equals the oracle on random distributed layouts;
* the oracle is pinned by the no-op property itself: every hardware index
  keeps its value, i.e. the output layout's coordinates are the operation
  applied to the input layout's coordinates (checked point by point);
* closure: distributed in, distributed out;
* reading A22: the packed mxfp4 A-fragment layout of config 5 is the bf16
  m16n8k16 A fragment after reshape k -> (kb, nibble) and split.
"""

import random

import pytest

import paper_2505_23819_b200 as ll
from oracle import f2
from oracle import shapeops as so
from oracle.constructors import mma_tile
from oracle.layout import Layout as OL
from workloads import configs


def rand_dist(rng, out_dims, zeros=0):
    d = sum(b for _, b in out_dims)
    n = d + zeros
    nreg = rng.randint(0, min(4, n))
    nlane = min(5, n - nreg)
    nw = n - nreg - nlane
    cols = [1 << k for k in range(d)] + [0] * zeros
    rng.shuffle(cols)
    tmp = OL([], out_dims, {})
    dims = [("reg", nreg), ("lane", nlane), ("warp", nw)]
    bases, k = {}, 0
    for nm, b in dims:
        bases[nm] = [tmp.unflatten(c) for c in cols[k:k + b]]
        k += b
    return OL(dims, out_dims, bases)


def to_ll(O):
    return ll.Layout(O.in_dims, O.out_dims, O.bases)


def from_ll(L):
    s = L.spec()
    return OL(s["in_dims"], s["out_dims"], s["bases"])


def points(L):
    """All hardware points as dicts."""
    res = []
    for h in range(1 << L.in_bits):
        pt, off = {}, 0
        for n, b in L.in_dims:
            pt[n] = (h >> off) & ((1 << b) - 1)
            off += b
        res.append(pt)
    return res


def test_trans_reshape_expand():
    rng = random.Random(1)
    for _ in range(40):
        L = rand_dist(rng, [("a", 2), ("b", 3), ("c", 2)], zeros=rng.randint(0, 1))
        perm = [2, 0, 1]
        O = so.trans(L, perm)
        assert from_ll(ll.transpose(to_ll(L), perm)) == O
        for pt in points(L):
            x = L.apply(pt)
            assert O.apply(pt) == tuple(x[p] for p in perm)       # no-op: same value
        R = so.reshape(L, [("p", 4), ("q", 3)])
        assert from_ll(ll.reshape(to_ll(L), [("p", 4), ("q", 3)])) == R
        for pt in points(L):
            assert R.flatten(R.apply(pt)) == L.flatten(L.apply(pt))
        E = so.expand_dims(L, 1, "e")
        assert from_ll(ll.expand_dims(to_ll(L), 1, "e")) == E
        for pt in points(L):
            x = L.apply(pt)
            assert E.apply(pt) == (x[0], 0) + tuple(x[1:])
        for X in (O, R, E):
            assert X.is_distributed()


def test_broadcast_uses_copies_then_registers():
    rng = random.Random(2)
    for zeros, bits in ((2, 2), (1, 3), (0, 1)):
        L = rand_dist(rng, [("a", 3), ("s", 0), ("c", 2)], zeros=zeros)
        B = so.broadcast(L, 1, bits)
        assert from_ll(ll.broadcast(to_ll(L), 1, bits)) == B
        assert B.is_distributed() and B.out_dims[1] == ("s", bits)
        for pt in points(L):
            x = L.apply(pt)
            y = B.apply(pt) if B.in_dims == L.in_dims else None
            if y is not None:
                assert (y[0], y[2]) == (x[0], x[2])                # other coords unchanged
        assert B.in_bits == L.in_bits + max(0, bits - zeros)


def test_join_split_round_trip():
    rng = random.Random(3)
    for _ in range(30):
        L = rand_dist(rng, [("a", 3), ("b", 3)], zeros=rng.randint(0, 1))
        J = so.join(L, "t")
        assert from_ll(ll.join(to_ll(L), "t")) == J
        # the two joined values of a hardware index sit in adjacent registers
        for pt in points(L):
            pt0 = dict(pt)
            pt0["reg"] = pt.get("reg", 0) << 1
            pt1 = dict(pt0)
            pt1["reg"] |= 1
            assert J.apply(pt0) == L.apply(pt) + (0,)
            assert J.apply(pt1) == L.apply(pt) + (1,)
        S = so.split(J)
        assert S == L and from_ll(ll.split(to_ll(J))) == L
        assert J.is_distributed() == L.is_distributed()


def test_split_rejects_non_register_dim():
    L = OL([("reg", 1), ("lane", 2)], [("a", 2), ("t", 1)],
           {"reg": [(1, 0)], "lane": [(2, 0), (0, 1)]})
    with pytest.raises(ValueError):
        so.split(L)
    with pytest.raises(ll.LLError) as e:
        ll.split(to_ll(L))
    assert e.value.name == "LL_ERR_UNSUPPORTED"


def test_config5_packed_layout_from_shape_ops_reading_A22():
    """The bf16 m16n8k16 A fragment (PTX formula, oracle constructor) tiled over
    a 128 x 128 (m, k) block, then reshape k -> (kb, nibble) and split: the
    packed-byte layout of config 5's destination (reading A22)."""
    frag = mma_tile("lhs", 16)                     # reg [k0, m3, k3], lane [k1, k2, m0, m1, m2]
    # element layout over (m: 7 bits, k: 7 bits): the fragment + register
    # repeats along k (k4, k5, k6) and m (m6), warps along m (m4, m5)
    spec = {"in_dims": [("reg", 7), ("lane", 5), ("warp", 2)], "out_dims": [("m", 7), ("k", 7)],
            "bases": {"reg": [(0, 1), (8, 0), (0, 8), (0, 16), (0, 32), (0, 64), (64, 0)],
                      "lane": [(0, 2), (0, 4), (1, 0), (2, 0), (4, 0)],
                      "warp": [(16, 0), (32, 0)]}}
    E = OL(**spec)
    # its first 3 reg bits and the lanes are exactly the PTX fragment
    assert [E.bases["reg"][i] for i in range(3)] == [tuple(v) for v in frag.bases["reg"]]
    assert [tuple(v) for v in E.bases["lane"]] == [tuple(v) for v in frag.bases["lane"]]
    P = so.split(so.reshape(E, [("m", 7), ("kb", 6), ("nib", 1)]))
    want = configs.cfg5(m_bits=7, kb_bits=6)["B"]
    W = OL(want["in_dims"], want["out_dims"], want["bases"])    # (with an empty block dim)
    assert P.out_dims == W.out_dims and P.cols == W.cols
    assert [(n, b) for n, b in W.in_dims if b] == P.in_dims
    # same through the C ABI
    Q = ll.split(ll.reshape(ll.Layout(**spec), [("m", 7), ("kb", 6), ("nib", 1)]))
    assert from_ll(Q) == P


# --- sliced layouts and the layout constructors --------

def _blocked_cases():
    from oracle.constructors import blocked
    return [
        (blocked([4, 5], [0, 3], [2, 2], [2, 0], [1, 0]), 1),
        (blocked([4, 5], [0, 3], [2, 2], [2, 0], [1, 0]), 0),
        (blocked([3, 4, 2], [1, 1, 1], [1, 3, 1], [1, 0, 0], [2, 1, 0]), 1),
    ]


def test_oracle_slice_removes_rows_and_keeps_surjectivity():
    """the slice removes the dim's rows; columns become zero exactly
    where the layout reached only that dim; the result is surjective (and, for
    these one-hot blocked layouts, has as many zero columns as the dim had
    bits)."""
    from oracle import shapeops
    for L, ax in _blocked_cases():
        S = shapeops.slice_(L, ax)
        dbits = L.out_dims[ax][1]
        assert S.out_bits == L.out_bits - dbits
        assert S.is_surjective()
        zero = [c for c in S.cols if c == 0]
        assert len(zero) == dbits
        # every hardware index holds the reduction-result index of its element:
        # the coordinates of L(h) other than `ax` (brute force over all h)
        for h in range(1 << L.in_bits):
            full = L.unflatten(L.apply_flat(h))
            assert S.unflatten(S.apply_flat(h)) == tuple(c for i, c in enumerate(full) if i != ax)


def test_ll_slice_blocked_mma_match_oracle():
    """C ABI constructors (ll_blocked, ll_mma_tile, ll_slice) agree with the
    oracle's (written separately from the paper)."""
    import paper_2505_23819_b200 as ll
    from oracle import shapeops
    from oracle.constructors import blocked, mma_tile

    def same(a_ll, b_or):
        sp = a_ll.spec()
        return (sp["in_dims"] == b_or.in_dims and sp["out_dims"] == b_or.out_dims and
                all(list(map(tuple, sp["bases"][n])) == list(b_or.bases[n]) for n, _ in b_or.in_dims))

    for args in (([4, 5], [0, 3], [2, 2], [2, 0], [1, 0]), ([3, 4, 2], [1, 1, 1], [1, 3, 1], [1, 0, 0], [2, 1, 0]),
                 ([7, 7], [0, 3], [2, 3], [5, 1], [1, 0])):
        B_ll, B_or = ll.blocked(*args), blocked(*args)
        assert same(B_ll, B_or), args
        for ax in range(len(args[0])):
            assert same(ll.slice_layout(B_ll, ax), shapeops.slice_(B_or, ax))
    for op in ("lhs", "rhs", "out"):
        for b in (8, 16, 32):
            assert same(ll.mma_tile(op, b), mma_tile(op, b)), (op, b)
    with pytest.raises(ll.LLError):
        ll.blocked([4], [1], [1], [1], [0])          # 1 + 1 + 1 != 4
