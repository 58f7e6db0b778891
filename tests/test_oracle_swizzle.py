"""Oracle pins: bank counter, optimal swizzling, warp-shuffle plans (CPU)."""

import random

import pytest

from oracle import banks, f2, shuffle, swizzle
from oracle.layout import Layout, from_flat
from workloads import configs
from tests.conftest import golden_rows


def L_from_spec(s):
    return Layout(s["in_dims"], s["out_dims"], s["bases"])


def rand_dist(rng, d, nreg, nlane=5):
    cols = [1 << k for k in range(d)]
    rng.shuffle(cols)
    nw = d - nreg - nlane
    cs = [(c,) for c in cols]
    return Layout([("reg", nreg), ("lane", nlane), ("warp", nw)], [("t", d)],
                  {"reg": cs[:nreg], "lane": cs[nreg:nreg + nlane], "warp": cs[nreg + nlane:]})


def warp_tile(L):
    """The warp-0 part of a layout with block bits (drop 'block')."""
    dims = [(n, b) for n, b in L.in_dims if n != "block"]
    used = set()
    for n, _ in dims:
        for v in L.bases[n]:
            used.add(L.flatten(v))
    # compress the tensor onto the bits the tile uses
    bits = sorted(x.bit_length() - 1 for x in used if x)
    remap = {1 << b: 1 << k for k, b in enumerate(bits)}
    bases = {n: [(remap[L.flatten(v)],) for v in L.bases[n]] for n, _ in dims}
    return Layout(dims, [("t", len(bits))], bases)


# --------------------------------------------------------------- bank counter / lemma

@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_bank_lemma_matches_brute_force(w):
    """Appendix lemma: n.c wavefronts per instruction, n >= 1,
    with c from L_bank (reading A13) -- against the brute-force counter."""
    rng = random.Random(20 + w)
    checked = 0
    while checked < 40:
        d = rng.randint(8, 11)
        nreg = rng.randint(1, d - 6)
        L = rand_dist(rng, d, nreg)
        regs = L.sub("reg")
        vmax = max(0, min(nreg, {1: 4, 2: 3, 4: 2, 8: 1}[w]))
        v = rng.randint(0, vmax)
        if (1 << v) * w < 4:
            continue
        V = regs[:v]
        b = min(d - v, (128 // ((1 << v) * w)).bit_length() - 1)
        ell = d - v - b
        vmask = sum(V)
        cands = [x for x in range(1, 1 << d) if not x & vmask]   # aligned vector access
        idx = []
        while len(idx) < ell:
            x = rng.choice(cands)
            if not f2.in_span(x, V + idx):
                idx.append(x)
        bank = f2.complete_basis(V + idx, d)
        S = from_flat([("offset", d)], L.out_dims, V + bank + idx)
        total, per = banks.count_wavefronts(S, L, w, list(range(v)), per_instruction=True)
        lemma = banks.lemma_wavefronts_per_instruction(V, idx, L.sub("lane"), w)
        assert all(p == lemma for p in per), (per[:4], lemma)
        checked += 1


def test_bank_counter_simple_cases():
    """Unswizzled row-major 32x32 fp32 read by rows (1 wavefront per
    instruction) vs by columns (32-way conflict)."""
    out = [("i", 5), ("j", 5)]
    S = Layout([("offset", 10)], out, {"offset": [(0, 1 << k) for k in range(5)] +
                                                  [(1 << k, 0) for k in range(5)]})
    rows = Layout([("reg", 5), ("lane", 5)], out,
                  {"reg": [(1 << k, 0) for k in range(5)], "lane": [(0, 1 << k) for k in range(5)]})
    cols = Layout([("reg", 5), ("lane", 5)], out,
                  {"reg": [(0, 1 << k) for k in range(5)], "lane": [(1 << k, 0) for k in range(5)]})
    assert banks.count_wavefronts(S, rows, 4, []) == 32
    assert banks.count_wavefronts(S, cols, 4, []) == 32 * 32


# --------------------------------------------------------------- abstract lemma

def test_abstract_swizzling_lemma_brute_force():
    """the largest subspace meeting U u V only in 0 has dimension
    d - max(dim U, dim V) -- 120 random cases, brute force over subspaces."""
    rng = random.Random(30)
    for _ in range(120):
        d = rng.randint(1, 5)
        U = [rng.getrandbits(d) for _ in range(rng.randint(0, d))]
        V = [rng.getrandbits(d) for _ in range(rng.randint(0, d))]
        assert swizzle.brute_force_max_trivial_dim(U, V, d) == swizzle.abstract_lemma_dim(U, V, d)


# --------------------------------------------------------------- the construction

def _ideal(L, w, v):
    """n wavefronts per instruction when conflict-free (lemma with c = 1)."""
    n_instr = (1 << L.in_bits) // 32 // (1 << v)
    return n_instr * max(1, ((1 << v) * w) // 4)


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_optimal_swizzle_is_conflict_free_random_pairs(w):
    """P:713 "M is the swizzled layout that minimizes read and write bank
    conflicts": for random distributed pairs with granule >= 4 bytes, the
    construction (main-text rule, reading A13) gives the ideal n wavefronts
    per instruction on both sides, and its index dimension is the abstract
    lemma's bound."""
    rng = random.Random(40 + w)
    seen = 0
    tries = 0
    while seen < 25 and tries < 2000:
        tries += 1
        d = rng.randint(8, 11)
        nreg = rng.randint(2, d - 6)
        A, B = rand_dist(rng, d, nreg), rand_dist(rng, d, nreg)
        V = swizzle.vector_set(A, B, w)
        if (1 << len(V)) * w < 4:
            continue
        S, info = swizzle.optimal_swizzle(A, B, w, V=V)
        assert S.is_memory() or all(f2.popcount(c) >= 1 for c in S.cols)
        assert f2.rank(S.cols) == d
        U = V + info["A_bank"]
        W = V + info["B_bank"]
        assert len(info["H"]) + len(info["C"]) == swizzle.abstract_lemma_dim(U, W, d)
        wa, wb = swizzle.swizzle_wavefronts(S, A, B, w, V)
        if not info["unavoidable"]:
            assert wa == _ideal(A, w, len(V)) and wb == _ideal(B, w, len(V))
        seen += 1
    assert seen == 25


def test_optimal_swizzle_matches_brute_force_optimum():
    """Exhaustive search over index subspaces for tiny tensors: the paper's
    construction reaches the minimum total wavefronts."""
    rng = random.Random(50)
    for _ in range(12):
        d = 7
        A, B = rand_dist(rng, d, 2), rand_dist(rng, d, 2)
        V = swizzle.vector_set(A, B, 4)
        S, info = swizzle.optimal_swizzle(A, B, 4, V=V)
        wa, wb = swizzle.swizzle_wavefronts(S, A, B, 4, V)
        assert wa + wb == swizzle.brute_force_min_wavefronts(A, B, 4, V)


@pytest.mark.parametrize("variant", ["mma", "T"])
def test_config1_swizzle_ideal(variant):
    c = configs.cfg1(variant)
    A, B = L_from_spec(c["A"]), L_from_spec(c["B"])
    S, info = swizzle.optimal_swizzle(A, B, 2)
    V = info["V"]
    wa, wb = swizzle.swizzle_wavefronts(S, A, B, 2, V)
    assert len(V) == (1 if variant == "mma" else 2)
    assert wa == _ideal(A, 2, len(V)) and wb == _ideal(B, 2, len(V))


def test_config2_tile_swizzle_ideal():
    """cfg2 CTA tile (mma C -> blocked, 128x128 fp16): V = {j0, i3, j3}?  The
    paper's V = A_reg cap B_reg in A's order; conflict-free both sides."""
    c = configs.cfg2(batch_bits=0)
    A, B = warp_tile(L_from_spec(c["A"])), warp_tile(L_from_spec(c["B"]))
    S, info = swizzle.optimal_swizzle(A, B, 2)
    V = info["V"]
    assert (1 << len(V)) * 2 == 16
    wa, wb = swizzle.swizzle_wavefronts(S, A, B, 2, V)
    assert wa == _ideal(A, 2, len(V)) and wb == _ideal(B, 2, len(V))


def test_config5_tile_swizzle_ideal():
    c = configs.cfg5(m_bits=7, kb_bits=6)
    A, B = warp_tile(L_from_spec(c["A"])), warp_tile(L_from_spec(c["B"]))
    S, info = swizzle.optimal_swizzle(A, B, 1)
    V = info["V"]
    assert (1 << len(V)) == 8        # {kb2, kb3, m6}: 8 bytes
    wa, wb = swizzle.swizzle_wavefronts(S, A, B, 1, V)
    assert wa == _ideal(A, 1, len(V)) and wb == _ideal(B, 1, len(V))


def test_subword_granule_is_not_optimal_reading_A17():
    """Lemma case 'not enough vectorization': with 2-byte granules the
    construction can leave conflicts -- a 64x64 bf16 transpose, one element per
    access (v = 0), needs more write wavefronts than the ideal."""
    out = [("i", 6), ("j", 6)]
    def bit(n):
        return (1 << int(n[1:]), 0) if n[0] == "i" else (0, 1 << int(n[1:]))
    rowL = Layout([("reg", 3), ("lane", 5), ("warp", 4)], out,
                  {"reg": [bit(x) for x in ["i3", "i4", "i5"]],
                   "lane": [bit(x) for x in ["j0", "j1", "j2", "j3", "j4"]],
                   "warp": [bit(x) for x in ["j5", "i0", "i1", "i2"]]})
    colL = Layout([("reg", 3), ("lane", 5), ("warp", 4)], out,
                  {"reg": [bit(x) for x in ["j3", "j4", "j5"]],
                   "lane": [bit(x) for x in ["i0", "i1", "i2", "i3", "i4"]],
                   "warp": [bit(x) for x in ["i5", "j0", "j1", "j2"]]})
    S, info = swizzle.optimal_swizzle(rowL, colL, 2, V=[])
    wa, wb = swizzle.swizzle_wavefronts(S, rowL, colL, 2, [])
    n_instr = (1 << 12) // 32
    assert wa + wb > 2 * n_instr


# --------------------------------------------------------------- warp shuffles

def test_fig4_shuffle_example_reading_A9():
    g = {r[0]: r[1:] for r in golden_rows("fig4_shuffle.txt")}
    def vec(s):
        return sum(int(ch) << k for k, ch in enumerate(s))
    A = Layout([("reg", 1), ("lane", 2)], [("x", 3)], {"reg": [(4,)], "lane": [(1,), (2,)]})
    B = Layout([("reg", 1), ("lane", 2)], [("x", 3)], {"reg": [(1,)], "lane": [(4,), (2,)]})
    p = shuffle.shuffle_plan(A, B, 4)
    assert p["V"] == []
    assert sorted(f2.span(p["V"] + p["I"] + p["G"])) == sorted(vec(s) for s in g["span"])
    assert shuffle.round_set(p, 0) == set(f2.span(p["V"] + p["I"] + p["G"]))
    assert vec(g["R0"][0]) == 0
    assert p["R"] == [vec(g["R1_reading_A9"][0])]
    assert vec(g["R1_printed"][0]) in f2.span(p["V"] + p["I"] + p["G"])   # why A9 is needed
    assert p["rounds"] == int(g["rounds"][0])
    sim = shuffle.simulate(A, B, p)
    assert sim["ok"]


def test_shuffle_simulator_random_warp_local_pairs():
    """2^|R| rounds, each thread sends and receives exactly one vector per
    round, and the final registers hold B's placement."""
    rng = random.Random(60)
    for _ in range(100):
        nreg = rng.randint(1, 3)
        nlane = rng.randint(1, 5)
        d = nreg + nlane
        w = rng.choice([1, 2, 4])
        cols = [1 << k for k in range(d)]
        rng.shuffle(cols)
        A = Layout([("reg", nreg), ("lane", nlane)], [("t", d)],
                   {"reg": [(c,) for c in cols[:nreg]], "lane": [(c,) for c in cols[nreg:]]})
        rng.shuffle(cols)
        B = Layout([("reg", nreg), ("lane", nlane)], [("t", d)],
                   {"reg": [(c,) for c in cols[:nreg]], "lane": [(c,) for c in cols[nreg:]]})
        p = shuffle.shuffle_plan(A, B, w)
        assert len(p["R"]) == d - len(p["V"]) - len(p["I"]) - len(p["G"])
        sim = shuffle.simulate(A, B, p)
        assert sim["ok"], (A, B, p)


def test_shuffle_plan_preconditions():
    A = Layout([("reg", 1), ("lane", 1), ("warp", 1)], [("t", 3)],
               {"reg": [(1,)], "lane": [(2,)], "warp": [(4,)]})
    B = Layout([("reg", 1), ("lane", 1), ("warp", 1)], [("t", 3)],
               {"reg": [(4,)], "lane": [(2,)], "warp": [(1,)]})
    with pytest.raises(ValueError):
        shuffle.shuffle_plan(A, B, 4)


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("w", [1, 2, 4])
def test_tma_swizzle_modes_are_def5_instances(m, w):
    """The TMA tensor-copy swizzle modes (32/64/128 B: 16-byte chunk bits
    [4, 4+m) of the shared-memory byte address XOR-ed with bits [7, 7+m), the
    CUDA programming guide's pattern, written out here) place every element
    exactly where Def. 5 puts it with vec = 16 bytes,
    per_phase = 128 / row bytes and max_phase = row bytes / 16, rows of 16 << m
    bytes.  This is what lets the TMA-fed path (LL_PATH_SMEM_TMA) reason about
    the hardware's image with the paper's machinery."""
    from oracle.constructors import mma_swizzle_layout, mma_swizzle_offset
    row_bytes = 16 << m
    n = (row_bytes // w).bit_length() - 1          # column bits per row
    rows = 32
    vec, per_phase, max_phase = 16 // w, 128 // row_bytes, row_bytes // 16
    mask = (1 << m) - 1
    for i in range(rows):
        for j in range(1 << n):
            a = i * row_bytes + j * w                 # dense (unswizzled) byte address
            hw = a ^ (((a >> 7) & mask) << 4)          # hardware swizzle
            assert hw % w == 0
            assert hw // w == mma_swizzle_offset(i, j, n, vec, per_phase, max_phase), (i, j)
    # and the matrix form printed after Def. 5 maps each hardware offset back
    L = mma_swizzle_layout(5, n, vec, per_phase, max_phase)
    for i in range(rows):
        for j in range(1 << n):
            a = i * row_bytes + j * w
            hw = (a ^ (((a >> 7) & mask) << 4)) // w
            assert L.apply_flat(hw) == (i << n) | j
