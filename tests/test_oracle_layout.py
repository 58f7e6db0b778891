"""Oracle pins: F2 algebra, layouts and constructors (CPU only).

Each test pins the oracle to something other than itself: numbers printed in
the paper (tests/golden), closed forms, the PTX ISA fragment formulas, brute
force on tiny inputs, or invariants.
"""

import itertools
import random

import pytest

from oracle import f2
from oracle.constructors import (blocked, identity, mma_swizzle_layout, mma_swizzle_offset,
                                 mma_tile)
from oracle.layout import (Layout, compose, from_flat, left_divide, product, right_inverse)
from workloads import configs
from tests.conftest import golden_rows


def L_from_spec(s):
    return Layout(s["in_dims"], s["out_dims"], s["bases"])


def layout_A():
    return blocked([4, 4], R=[1, 1], T=[2, 3], W=[1, 0], order=[1, 0])


# ---------------------------------------------------------------------------- paper pins

def test_matrix_A_bits_match_paper():
    """P:283-295 displays A bit by bit; the blocked constructor (Appendix proof,
    P:1011-1025) with 2x2 regs, 4x8 threads, 2x1 warps must give it."""
    rows = [[int(x) for x in r] for r in golden_rows("matrix_A.txt")]
    A = layout_A()
    cols = A.cols
    assert len(cols) == 8
    for r in range(8):
        for c in range(8):
            assert (cols[c] >> r) & 1 == rows[r][c], (r, c)
    # and the workload table used for config 1 is the same matrix
    assert L_from_spec(configs.cfg1()["A"]).cols == cols


def test_tab_mapping_rows():
    """tab:mapping: ten printed location <-> (reg, thread, warp) rows."""
    A = layout_A()
    for i, j, r, t, w in golden_rows("tab_mapping.txt"):
        assert A.apply({"reg": int(r), "lane": int(t), "warp": int(w)}) == (int(i), int(j))


def test_worked_example_t9_r1():
    """P:274-277 / P:305-306: r1 of t9 of w0 is at (2, 3); and it is the XOR of
    the per-level locations (0,1) xor (2,2) xor (0,0)."""
    (r, t, w, i, j), = golden_rows("worked_example.txt")
    A = layout_A()
    assert A.apply({"reg": int(r), "lane": int(t), "warp": int(w)}) == (int(i), int(j))
    assert A.apply({"reg": 1}) == (0, 1)
    assert A.apply({"lane": 9}) == (2, 2)
    # w_j = [1 1 0 0]^T = 3, w_i = [0 1 0 0]^T = 2
    v = 1 | (9 << 2)
    assert f2.apply(A.cols, v) == (2 << 4) | 3


def test_matrix_A_is_distributed_and_bijective():
    A = layout_A()
    assert A.is_distributed() and A.is_surjective()
    assert sorted(f2.apply(A.cols, h) for h in range(256)) == list(range(256))


# ---------------------------------------------------------------------- F2 algebra

def rand_matrix(rng, m, n):
    return [rng.getrandbits(m) for _ in range(n)]


def test_matmul_by_hand_and_associativity():
    # [[1,0],[1,1]] x [[1,1],[0,1]] = [[1,1],[1,0]]  (columns: LSB = row 0)
    a = [0b11, 0b10]
    b = [0b01, 0b11]
    assert f2.matmul(a, b) == [0b11, 0b01]
    rng = random.Random(1)
    for _ in range(200):
        m, n, p, q = (rng.randint(1, 12) for _ in range(4))
        A, B, C = rand_matrix(rng, m, n), rand_matrix(rng, n, p), rand_matrix(rng, p, q)
        assert f2.matmul(f2.matmul(A, B), C) == f2.matmul(A, f2.matmul(B, C))


def test_rank_against_brute_force():
    rng = random.Random(2)
    for _ in range(300):
        d = rng.randint(1, 6)
        vecs = [rng.getrandbits(d) for _ in range(rng.randint(0, 6))]
        assert (1 << f2.rank(vecs)) == len(f2.span(vecs))


def test_right_inverse_is_right_inverse():
    """M M^{-1} = I for surjective M."""
    rng = random.Random(3)
    done = 0
    while done < 300:
        m, n = rng.randint(1, 10), rng.randint(1, 14)
        M = rand_matrix(rng, m, n)
        if f2.rank(M) < m:
            with pytest.raises(ValueError):
                f2.right_inverse(M, m)
            continue
        X = f2.right_inverse(M, m)
        assert f2.matmul(M, X) == [1 << i for i in range(m)]
        done += 1


def test_right_inverse_by_hand():
    # [1 1] (1x2) -> [1, 0]^T: the slack variable is zero
    assert f2.right_inverse([1, 1], 1) == [0b01]
    # a permutation matrix inverts to its transpose
    A = layout_A()
    X = f2.right_inverse(A.cols, 8)
    for r in range(8):
        for c in range(8):
            assert (X[c] >> r) & 1 == (A.cols[r] >> c) & 1


def test_min_weight_on_broadcast_layouts():
    """with zero / duplicated-source columns, free variables set to
    zero give a minimum-Hamming-weight solution; brute force over <= 6 free bits
    for distributed layouts with broadcast (zero) columns."""
    rng = random.Random(4)
    for _ in range(200):
        d = rng.randint(1, 5)
        extra = rng.randint(0, 4)
        cols = [1 << k for k in range(d)] + [0] * extra
        rng.shuffle(cols)
        X = f2.right_inverse(cols, d)
        for t in range(d):
            sols = f2.solve_all(cols, 1 << t)
            best = min(f2.popcount(s) for s in sols)
            assert f2.popcount(X[t]) == best
            assert X[t] == min(sols)          # lowest preimage (reading A4)


def test_complete_basis():
    assert f2.complete_basis([], 2) == [1, 2]
    assert f2.complete_basis([0b101], 3) == [1, 2]
    assert f2.complete_basis([1, 2, 4], 3) == []
    with pytest.raises(ValueError):
        f2.complete_basis([3, 3], 3)


def test_intersection_dim_brute_force():
    rng = random.Random(5)
    for _ in range(300):
        d = rng.randint(1, 6)
        U = [rng.getrandbits(d) for _ in range(rng.randint(0, 4))]
        V = [rng.getrandbits(d) for _ in range(rng.randint(0, 4))]
        inter = f2.span(U) & f2.span(V)
        assert (1 << f2.intersection_dim(U, V)) == len(inter)


# ---------------------------------------------------------------------- layout ops

def rand_distributed(rng, d, nreg, nlane, nwarp, zeros=0):
    cols = [1 << k for k in range(d)] + [0] * zeros
    rng.shuffle(cols)
    nb = len(cols)
    assert nreg + nlane + nwarp == nb
    cs = [(c,) for c in cols]
    return Layout([("reg", nreg), ("lane", nlane), ("warp", nwarp)], [("t", d)],
                  {"reg": cs[:nreg], "lane": cs[nreg:nreg + nlane], "warp": cs[nreg + nlane:]})


def test_compose_with_inverse_is_identity_off_the_kernel():
    rng = random.Random(6)
    for _ in range(100):
        d = rng.randint(2, 8)
        L = rand_distributed(rng, d, 1, d - 2, 1) if d >= 2 else None
        inv = right_inverse(L)
        LL = compose(L, inv)            # L o L^{-1} = id on the tensor
        assert LL.cols == [1 << k for k in range(d)]
        back = compose(inv, L)          # L^{-1} o L = id (bijective L)
        assert back.cols == [1 << k for k in range(d)]


def test_product_and_left_divide_round_trip():
    """Definitions Product and Left Division."""
    rng = random.Random(7)
    for _ in range(100):
        a = rng.randint(1, 3)
        b = rng.randint(1, 3)
        M1 = Layout([("reg", a)], [("x", a)], {"reg": [(rng.getrandbits(a),) for _ in range(a)]})
        M2 = Layout([("reg", b)], [("x", b)], {"reg": [(rng.getrandbits(b),) for _ in range(b)]})
        M = product(M1, M2)
        assert M.in_dims == [("reg", a + b)] and M.out_dims == [("x", a + b)]
        assert left_divide(M, M1) == M2
    # off-diagonal one -> not divisible  ([[1,1],[0,1]] / [1])
    M = Layout([("reg", 2)], [("x", 2)], {"reg": [(1,), (3,)]})
    with pytest.raises(ValueError):
        left_divide(M, Layout([("reg", 1)], [("x", 1)], {"reg": [(1,)]}))


def test_identity_and_product_build_matrix_A():
    """The Appendix construction as an explicit product of identity tiles."""
    parts = [identity(1, "reg", "dim1"), identity(1, "reg", "dim0"), identity(3, "lane", "dim1"),
             identity(2, "lane", "dim0"), identity(1, "warp", "dim0")]
    L = parts[0]
    for p in parts[1:]:
        L = product(L, p)
    from oracle.layout import with_out_order
    L = with_out_order(L, ["dim0", "dim1"])
    assert L.cols == layout_A().cols


def test_broadcast_mask():
    A = layout_A()
    assert A.broadcast_mask("reg") == 0
    Ab = product(A, Layout([("reg", 1)], [], {"reg": [()]}))
    assert Ab.broadcast_mask("reg") == 0b100          # registers 4-7 repeat 0-3
    assert Ab.is_distributed()
    dup = Layout([("reg", 2)], [("x", 1)], {"reg": [(1,), (1,)]})
    assert not dup.is_distributed()


# --------------------------------------------------------------- mma tiles vs PTX ISA

def ptx_A_fragment(bits, lane, e):
    """PTX ISA 'Matrix fragments for mma.m16n8k{8,16,32}' A operand (row, col)."""
    g, t = lane >> 2, lane & 3
    if bits == 16:      # m16n8k16 .f16/.bf16: a0..a7
        return g + 8 * ((e >> 1) & 1), t * 2 + (e & 1) + 8 * (e >> 2)
    if bits == 8:       # m16n8k32 .s8/.e4m3: a0..a15
        return g + 8 * ((e >> 2) & 1), t * 4 + (e & 3) + 16 * (e >> 3)
    if bits == 32:      # m16n8k8 .tf32: a0..a3
        return g + 8 * (e & 1), t + 4 * (e >> 1)
    raise ValueError


def ptx_B_fragment16(lane, e):
    """m16n8k16 B operand b0..b3: (row = k, col = n)."""
    g, t = lane >> 2, lane & 3
    return t * 2 + (e & 1) + 8 * (e >> 1), g


def ptx_C_fragment(lane, e):
    """m16n8 accumulator c0..c3: (row, col)."""
    g, t = lane >> 2, lane & 3
    return g + 8 * (e >> 1), t * 2 + (e & 1)


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_mma_lhs_tile_matches_ptx(bits):
    L = mma_tile("lhs", bits)
    n = 1 << L.in_size("reg")
    assert n == {8: 16, 16: 8, 32: 4}[bits]
    for lane in range(32):
        for e in range(n):
            assert L.apply({"reg": e, "lane": lane}) == ptx_A_fragment(bits, lane, e)


def test_mma_rhs_tile_reading_A8():
    L = mma_tile("rhs", 16)
    for lane in range(32):
        for e in range(4):
            assert L.apply({"reg": e, "lane": lane}) == ptx_B_fragment16(lane, e)
    # the literal printed formula places reg bit 1 on n3 (a k8 x n16 tile): not PTX
    P = mma_tile("rhs", 16, rhs_reading="printed")
    assert any(P.apply({"reg": e, "lane": l}) != ptx_B_fragment16(l, e)
               for l in range(32) for e in range(4))


def test_mma_out_tile_matches_ptx_and_config_tables():
    L = mma_tile("out", 16)
    for lane in range(32):
        for e in range(4):
            assert L.apply({"reg": e, "lane": lane}) == ptx_C_fragment(lane, e)
    # config 2's A = C tile x id^{reg,1}_4 x id^{reg,0}_1 x id^{warp,0}_2 x block
    from oracle.layout import with_out_order
    T = product(L, identity(4, "reg", "dim1"))
    T = product(T, identity(1, "reg", "dim0"))
    T = product(T, identity(2, "warp", "dim0"))
    T = with_out_order(T, ["dim0", "dim1"])
    A2 = L_from_spec(configs.cfg2(batch_bits=0)["A"])
    assert [c for c in T.cols] == A2.cols[:len(T.cols)]
    # config 1a's B: the C tile over two warps along j
    B1 = L_from_spec(configs.cfg1("mma")["B"])
    T1 = with_out_order(product(L, identity(1, "warp", "dim1")), ["dim0", "dim1"])
    assert T1.cols == B1.cols


def test_config2_B_is_blocked_tile_times_register_repeats():
    """blocked sizePerThread [1,8], threadsPerWarp [2,16], warpsPerCTA [4,1]
     on an 8x128 tile, repeated over registers along dim 0."""
    from oracle.layout import with_out_order
    T = blocked([3, 7], R=[0, 3], T=[1, 4], W=[2, 0], order=[1, 0])
    T = with_out_order(product(T, identity(4, "reg", "dim0")), ["dim0", "dim1"])
    B2 = L_from_spec(configs.cfg2(batch_bits=0)["B"])
    assert T.cols == B2.cols


def test_config5_A_is_blocked():
    from oracle.layout import with_out_order
    T = blocked([5, 6], R=[0, 4], T=[3, 2], W=[2, 0], order=[1, 0])
    T = with_out_order(product(T, identity(2, "reg", "dim0")), ["dim0", "dim1"])
    A5 = L_from_spec(configs.cfg5(m_bits=7, kb_bits=6)["A"])
    assert T.cols == A5.cols


def test_config5_B_is_packed_A_fragment():
    """Reading A22: bf16 m16n8k16 A fragment on a 128 x 128(k) tile with the
    k0 nibble bit removed (kb = k >> 1); checked element by element against the
    PTX A-fragment formula."""
    B5 = L_from_spec(configs.cfg5(m_bits=7, kb_bits=6)["B"])
    # B5 reg bits: [m3, kb2, kb3, kb4, kb5, m6]; lane [kb0, kb1, m0, m1, m2]; warp [m4, m5]
    for lane in range(32):
        for e in range(8):
            r, k = ptx_A_fragment(16, lane, e)
            if k & 1:
                continue                     # the nibble partner shares the byte
            kb = k >> 1
            # PTX element e: bit1 -> m3, bit2 -> k3 (= kb2); lane bits as PTX
            reg = ((e >> 1) & 1) | (((e >> 2) & 1) << 1)
            assert B5.apply({"reg": reg, "lane": lane}) == (r, kb)


# ------------------------------------------------------------------- Def. 5 swizzling

def test_def5_matrix_structure_matches_formula_exhaustively():
    """Two statements of the paper pinned against each other: the Def. 5 formula
     and the [[I_n, C],[0, I_m]] structure with c_k (reading
    A7: c_k is the k-th column).  Exhaustive for m, n <= 4."""
    for m, n in itertools.product(range(1, 5), range(1, 5)):
        for vec in (1, 2, 4, 8):
            for pp in (1, 2, 4):
                for mp in (1, 2, 4, 8):
                    S = mma_swizzle_layout(m, n, vec, pp, mp)
                    assert S.is_memory() or (S.cols == [1 << k for k in range(m + n)])
                    for i in range(1 << m):
                        for j in range(1 << n):
                            off = mma_swizzle_offset(i, j, n, vec, pp, mp)
                            assert f2.apply(S.cols, off) == (i << n) | j


def test_def5_spec_example_and_involution():
    # SPEC-derived example: vec=2, per_phase=1, max_phase=2, m=1, n=2: (1,0) -> 6
    assert mma_swizzle_offset(1, 0, 2, 2, 1, 2) == 6
    S = mma_swizzle_layout(3, 4, 2, 1, 4)
    assert f2.matmul(S.cols, S.cols) == [1 << k for k in range(7)]       # M^2 = I
    assert mma_swizzle_layout(3, 4, 2, 1, 1).cols == [1 << k for k in range(7)]


def test_memory_layout_predicate():
    S = mma_swizzle_layout(3, 3, 1, 1, 8)
    assert S.is_memory()
    bad = Layout([("offset", 2)], [("x", 2)], {"offset": [(1,), (1,)]})
    assert not bad.is_memory()


def test_from_flat_round_trip():
    A = layout_A()
    B = from_flat(A.in_dims, A.out_dims, A.cols)
    assert B == A


def test_b8_matrix_tiles_measured_on_b200_are_linear_layouts():
    """sm_100a's 8-bit ldmatrix / stmatrix forms are linear layouts (the
    paper's claim for the 16-bit ones): the per-(lane, byte)
    shared-memory offsets measured on the B200 by tools/b8_probe.cu
    (profiles/r01/b8/b8_probe.json) equal apply() of the F2 layouts
      ldmatrix.m16n16.x1.trans.b8: reg [16, 32, 8], lane [64, 128, 1, 2, 4]
      stmatrix.m16n8.x1.trans.b8:  reg [16, 8],     lane [32, 64, 1, 2, 4]
    at every one of the 256 / 128 bytes (the tiles the register-faithful path
    would left-divide by; DESIGN 8b)."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "profiles", "r01", "b8", "b8_probe.json")
    d = json.load(open(p))
    ld = Layout([("reg", 3), ("lane", 5)], [("offset", 8)],
                {"reg": [(16,), (32,), (8,)], "lane": [(64,), (128,), (1,), (2,), (4,)]})
    got = d["ldmatrix.m16n16.x1.trans.b8"]
    for lane in range(32):
        for b in range(8):
            assert ld.apply({"reg": b, "lane": lane}) == (got[lane][b],)
    st = Layout([("reg", 2), ("lane", 5)], [("offset", 7)],
                {"reg": [(16,), (8,)], "lane": [(32,), (64,), (1,), (2,), (4,)]})
    mem = d["stmatrix.m16n8.x1.trans.b8"]
    for lane in range(32):
        for b in range(4):
            (o,) = st.apply({"reg": b, "lane": lane})
            assert mem[o] == (lane << 2) | b
    assert sum(v != 255 for v in mem) == 128
