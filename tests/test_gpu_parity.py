"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, byte-exact.

Inputs are seeded splitmix64 patterns (workloads.values) generated on the
device; expected outputs come only from ``oracle`` (plain definition of the
conversion / gather).  Buffers are compared as raw
bytes.  Small sizes: every element; full BASELINE sizes: sampled outputs
computed one by one by the oracle + a permutation property on the whole
buffer.
"""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import convert as oconv
from oracle import f2
from oracle.layout import Layout as OLayout
from workloads import configs
from workloads.values import indices_torch, values_torch

if torch.cuda.is_available():
    import paper_2505_23819_b200 as ll

_NP = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


def _olayout(spec):
    return OLayout(spec["in_dims"], spec["out_dims"], spec["bases"])


def _np(t, w):
    return t.cpu().numpy().view(_NP[w])


def run_convert(c, path="auto", batch=1, seed=7):
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    nA, nB = A.in_bits, B.in_bits
    src = values_torch((1 << nA) * batch, seed, w, "cuda")
    dst = torch.full(((1 << nB) * batch,), 0x55 if w == 1 else 0x5555, dtype=src.dtype, device="cuda") \
        if w <= 2 else torch.zeros((1 << nB) * batch, dtype=src.dtype, device="cuda")
    ll.convert(src, A, dst, B, 8 * w, path=path, batch=batch)
    torch.cuda.synchronize()
    return _np(src, w), _np(dst, w)


def expect_convert(c, src_np, batch=1):
    Ao, Bo = _olayout(c["A"]), _olayout(c["B"])
    nA, nB = Ao.in_bits, Bo.in_bits
    out = []
    for b in range(batch):
        out.append(oconv.convert_np(src_np[b << nA:(b + 1) << nA], Ao, Bo))
    return np.concatenate(out)


CASES = [
    ("cfg1a", lambda: configs.cfg1("mma")),
    ("cfg1b", lambda: configs.cfg1("T")),
    ("cfg2_b0", lambda: configs.cfg2(batch_bits=0)),
    ("cfg2_b3", lambda: configs.cfg2(batch_bits=3)),
    ("cfg3_64", lambda: configs.cfg3(n_bits=6)),
    ("cfg3_512", lambda: configs.cfg3(n_bits=9)),
    ("cfg3_rect", lambda: configs.cfg3(n_bits=9, m_bits=7)),
    ("cfg5_small", lambda: configs.cfg5(m_bits=8, kb_bits=7)),
    ("cfg5_mid", lambda: configs.cfg5(m_bits=9, kb_bits=9)),
    ("cfg6_small", lambda: configs.cfg6(n_bits=7, k_bits=7)),
    ("cfg6_rect", lambda: configs.cfg6(n_bits=6, k_bits=9)),
]


@pytest.mark.parametrize("path", ["auto", "smem", "smem_noswizzle", "smem_padded", "shuffle",
                                  "smem_async", "smem_tma", "smem_tma_store", "generic"])
@pytest.mark.parametrize("name,mk", CASES)
def test_convert_configs_small(name, mk, path):
    c = mk()
    if path == "shuffle" and name.startswith("cfg3"):
        pytest.skip("transpose exchange is not warp-local (P:624); covered by test_shuffle_rejects")
    if path in ("smem_async", "smem_tma", "smem_tma_store") and name.startswith("cfg1"):
        pytest.skip("16x16 tensor is smaller than one async tile")
    src, dst = run_convert(c, path=path)
    exp = expect_convert(c, src)
    assert dst.tobytes() == exp.tobytes()


@pytest.mark.parametrize("batch", [1, 5, 37])
def test_convert_ragged_batch(batch):
    """Batch of independent layout instances not a multiple of anything (the
    tail of the persistent grid)."""
    c = configs.cfg2(batch_bits=0)
    src, dst = run_convert(c, batch=batch, seed=11)
    assert dst.tobytes() == expect_convert(c, src, batch).tobytes()


def rand_pair(rng, d, w):
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    names = [("reg", rng.randint(vb, vb + 2)), ("lane", 5)]
    rest = d - names[0][1] - 5
    nw = min(rest, rng.randint(0, 3))
    names += [("warp", nw), ("block", rest - nw)]
    out = [("i", d // 2), ("j", d - d // 2)]
    tmp = OLayout([], out, {})
    specs = []
    for _ in range(2):
        cols = [1 << k for k in range(d)]
        rng.shuffle(cols)
        bases, k = {}, 0
        for n, b in names:
            bases[n] = [tmp.unflatten(x) for x in cols[k:k + b]]
            k += b
        specs.append({"in_dims": names, "out_dims": out, "bases": bases})
    return {"A": specs[0], "B": specs[1], "elem_bytes": w}


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_random_pairs(w):
    rng = random.Random(300 + w)
    for _ in range(15):
        d = rng.randint(12, 16)
        c = rand_pair(rng, d, w)
        src, dst = run_convert(c, seed=rng.randint(0, 1000))
        assert dst.tobytes() == expect_convert(c, src).tobytes()


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_vec32(w):
    """Knob vec32: 32-byte thread vectors (sm_100 256-bit LDG / STG) on the
    compiled smem kernel -- random pairs and the config families, byte-exact."""
    ll.tune("vec32", 1)
    try:
        rng = random.Random(350 + w)
        for _ in range(10):
            c = rand_pair(rng, rng.randint(12, 16), w)
            src, dst = run_convert(c, seed=rng.randint(0, 1000))
            assert dst.tobytes() == expect_convert(c, src).tobytes()
        for name, mk in CASES:
            c = mk()
            if c["elem_bytes"] != w and not (w == 2 and c["elem_bytes"] == 2):
                continue
            src, dst = run_convert(c)
            assert dst.tobytes() == expect_convert(c, src).tobytes(), name
    finally:
        ll.tune("vec32", 0)


def b8_pair(rng, kind, nr=3, nw=1, nb=2):
    """fp8 pairs the sm_100a 8-bit matrix tiles serve (the tiles
    measured in test_b8_matrix_tiles_measured_on_b200_are_linear_layouts):
    kind "both": B's lanes 2..4 and its first word bit hold A's lanes 2..4 and
    A's byte bit 1 (stmatrix.b8 writes, ldmatrix.b8 reads); "st_vec": B's
    bytes are A's lanes 2, 3 (stmatrix.b8 writes, vector reads); "ld_vec":
    A's bytes are B's lanes 2, 3 (vector writes, ldmatrix.b8 reads).  One
    tensor dim of nr + 5 + nw + nb bits; blocks identical."""
    d = nr + 5 + nw
    bits = list(range(d))
    rng.shuffle(bits)
    blk = list(range(d, d + nb))

    def mk(reg, lane, warp):
        return {"in_dims": [("reg", nr), ("lane", 5), ("warp", nw), ("block", nb)],
                "out_dims": [("t", d + nb)],
                "bases": {"reg": [(1 << b,) for b in reg], "lane": [(1 << b,) for b in lane],
                          "warp": [(1 << b,) for b in warp], "block": [(1 << b,) for b in blk]}}

    if kind == "ld_vec":
        Br, Bl, Bw = bits[:nr], bits[nr:nr + 5], bits[nr + 5:]
        fixed = [Bl[2], Bl[3], Bl[4]] + ([Br[2]] if nr >= 4 else [])
        rest = [b for b in bits if b not in fixed]
        rng.shuffle(rest)
        a = fixed + rest
        return {"A": mk(a[:nr], a[nr:nr + 5], a[nr + 5:]), "B": mk(Br, Bl, Bw), "elem_bytes": 1}
    Ar, Al, Aw = bits[:nr], bits[nr:nr + 5], bits[nr + 5:]
    if kind == "both":
        rest = [b for b in bits if b not in (Al[2], Al[3], Al[4], Ar[1])]
        rng.shuffle(rest)
        Br = [rest[0], rest[1]] + rest[2:2 + nr - 3]
        Br.insert(rng.randint(2, nr - 1), Ar[1])      # any of B's word bits
        r2 = rest[2 + nr - 3:]
        Bl, Bw = [r2[0], r2[1], Al[2], Al[3], Al[4]], r2[2:]
    else:
        fixed = [Al[2], Al[3], Al[4], Ar[1]][:max(2, min(4, nr))]
        rest = [b for b in bits if b not in fixed]
        rng.shuffle(rest)
        b = fixed + rest
        Br, Bl, Bw = b[:nr], b[nr:nr + 5], b[nr + 5:]
    return {"A": mk(Ar, Al, Aw), "B": mk(Br, Bl, Bw), "elem_bytes": 1}


@pytest.mark.parametrize("kind", ["both", "st_vec", "ld_vec"])
def test_convert_regs_b8_tiles(kind):
    """Register-faithful fp8 conversions lowered with stmatrix.m16n8.trans.b8
    / ldmatrix.m16n16.trans.b8 (x1 / x2 / x4 by words per thread), against
    the oracle; with the b8 tiles off the same pairs have no regs plan or a
    vector one."""
    rng = random.Random({"both": 81, "st_vec": 82, "ld_vec": 83}[kind])
    done = 0
    for nr, nw in ((3, 0), (3, 1), (4, 1), (4, 2), (5, 1)):
        for _ in range(3):
            c = b8_pair(rng, kind, nr=nr, nw=nw)
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            try:
                d = ll.plan_describe(A, B, 8, "regs")
            except ll.LLError:
                continue
            assert "b8" in d["regs"]["write"] + d["regs"]["read"], d["regs"]
            for batch in (1, 3):
                src, dst = run_convert(c, path="regs", batch=batch, seed=rng.randint(0, 99))
                assert dst.tobytes() == expect_convert(c, src, batch).tobytes(), (kind, nr, nw, d["regs"])
            done += 1
    assert done >= 6


def perm_pair(rng, d, w, r, which):
    """A random distributed layout A and B = A with its `which` columns
    ("reg" or "lane") permuted: the pair differs only in register order (no
    exchange between threads) or only in lane order (warp-local,
    P:624)."""
    names = [("reg", r), ("lane", 5)]
    rest = d - r - 5
    nw = min(rest, rng.randint(0, 2))
    names += [("warp", nw), ("block", rest - nw)]
    out = [("i", d // 2), ("j", d - d // 2)]
    tmp = OLayout([], out, {})
    cols = [1 << k for k in range(d)]
    rng.shuffle(cols)
    bases, k = {}, 0
    for n, b in names:
        bases[n] = [tmp.unflatten(x) for x in cols[k:k + b]]
        k += b
    A = {"in_dims": names, "out_dims": out, "bases": bases}
    bb = dict(bases)
    p = list(bb[which])
    if len(p) < 2:
        raise ValueError("perm_pair: %s needs at least two columns to permute" % which)
    while p == bases[which]:
        rng.shuffle(p)
    bb[which] = p
    return {"A": A, "B": {"in_dims": names, "out_dims": out, "bases": bb}, "elem_bytes": w}


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_register_permutation_pairs(w):
    """Pairs that differ only in register order: LL_PATH_REGPERM (no STS /
    LDS, no shuffles) applies whenever the permuted chunk is <= 64 bytes;
    AUTO takes the smem plan when it exchanges >= 8-byte granules, else the
    warp-shuffle exchange where it applies (w <= 4), else the permutation
    (the measured rule); all byte-exact, also batched and sharded."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    rng = random.Random(1500 + w)
    took = 0
    for case in range(8):
        r = rng.randint(2, max(2, vb + (6 - vb if w == 1 else 2)))
        c = perm_pair(rng, rng.randint(12, 15), w, r, "reg")
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        d = ll.plan_describe(A, B, 8 * w)
        if (w << max(r, vb)) <= 64:
            g = ll.plan_describe(A, B, 8 * w, "smem")["granule_bytes"]
            try:
                shfl = w <= 4 and ll.plan_describe(A, B, 8 * w, "shuffle")["granule_bytes"] <= 4
            except ll.LLError:
                shfl = False
            want = "smem" if g >= 8 else ("shuffle" if shfl else "regperm")
            assert d["path"] == want, (r, g, d["path"])
        batch = 1 + 2 * (case % 2)
        src, dst = run_convert(c, seed=case, batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes()
        try:
            ll.plan_describe(A, B, 8 * w, "regperm")
        except ll.LLError:
            assert (w << max(r, vb)) > 64
            continue
        took += 1
        src, dst = run_convert(c, path="regperm", seed=case + 10, batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes()
        n = 1 << A.in_bits
        full = values_torch(n, 77, w, "cuda")
        parts = []
        for s_ in range(4):
            s0, s1, d0, d1 = ll.shard_describe(A, B, 8 * w, 4, s_, "regperm")
            dl = torch.empty(d1 - d0, dtype=torch.uint8, device="cuda")
            ll.convert_shard(full.view(torch.uint8)[s0:s1].clone(), A, dl, B, 8 * w, 4, s_, path="regperm")
            parts.append(dl)
        torch.cuda.synchronize()
        got = torch.cat(parts).cpu().numpy().view(_NP[w])
        assert got.tobytes() == expect_convert(c, _np(full, w)).tobytes()
    assert took >= 4


@pytest.mark.parametrize("w", [1, 2, 4])
def test_convert_lane_permutation_pairs(w):
    """Pairs that differ only in lane order (warp-local): AUTO, the
    warp-shuffle exchange and the smem exchange all byte-exact."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    rng = random.Random(1600 + w)
    for case in range(6):
        c = perm_pair(rng, rng.randint(12, 15), w, vb, "lane")
        for path in ("auto", "shuffle", "smem"):
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            try:
                ll.plan_describe(A, B, 8 * w, path)
            except ll.LLError:
                assert path == "shuffle"
                continue
            src, dst = run_convert(c, path=path, seed=case)
            assert dst.tobytes() == expect_convert(c, src).tobytes(), (case, path)


@pytest.mark.parametrize("w", [1, 2, 4])
def test_convert_random_pairs_shuffle(w):
    rng = random.Random(500 + w)
    done = 0
    while done < 10:
        d = rng.randint(11, 15)
        c = rand_pair(rng, d, w)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            ll.plan_describe(A, B, 8 * w, "shuffle")
        except ll.LLError:
            continue
        src, dst = run_convert(c, path="shuffle", seed=rng.randint(0, 1000))
        assert dst.tobytes() == expect_convert(c, src).tobytes()
        done += 1


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_random_pairs_async(w):
    rng = random.Random(600 + w)
    done = 0
    while done < 10:
        d = rng.randint(12, 16)
        c = rand_pair(rng, d, w)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            ll.plan_describe(A, B, 8 * w, "smem_async")
        except ll.LLError:
            continue
        src, dst = run_convert(c, path="smem_async", seed=rng.randint(0, 1000))
        assert dst.tobytes() == expect_convert(c, src).tobytes()
        done += 1


@pytest.mark.parametrize("batch", [3, 37])
def test_convert_async_ragged_batch(batch):
    c = configs.cfg2(batch_bits=0)
    src, dst = run_convert(c, path="smem_async", batch=batch, seed=17)
    assert dst.tobytes() == expect_convert(c, src, batch).tobytes()


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_random_pairs_tma(w):
    """TMA-fed path: random bit-permutation pairs (box dims, swizzle modes and
    reader lanes all chosen by the planner) against the oracle."""
    rng = random.Random(700 + w)
    done, tried = 0, 0
    modes = set()
    while done < 12 and tried < 200:
        tried += 1
        d = rng.randint(12, 17)
        c = rand_pair(rng, d, w)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            plan = ll.plan_describe(A, B, 8 * w, "smem_tma")
        except ll.LLError:
            continue
        modes.add(plan["tma"]["swizzle"])
        src, dst = run_convert(c, path="smem_tma", seed=rng.randint(0, 1000))
        assert dst.tobytes() == expect_convert(c, src).tobytes(), plan["tma"]
        done += 1
    assert done >= 6, (done, tried)


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_random_pairs_tma_store(w):
    """TMA load + TMA store path on random bit-permutation pairs."""
    rng = random.Random(900 + w)
    done, tried = 0, 0
    while done < 12 and tried < 200:
        tried += 1
        c = rand_pair(rng, rng.randint(12, 17), w)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            plan = ll.plan_describe(A, B, 8 * w, "smem_tma_store")
        except ll.LLError:
            continue
        batch = rng.choice([1, 2, 5])
        src, dst = run_convert(c, path="smem_tma_store", seed=rng.randint(0, 1000), batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes(), plan["tma"]
        done += 1
    assert done >= 6, (done, tried)


@pytest.mark.parametrize("path", ["smem_tma", "smem_tma_store"])
@pytest.mark.parametrize("knobs", [{"tma_jit": 0}, {"tmaj_tpc": -1}, {"tmaj_tpc": -1, "tmaj_stages": 3},
                                   {"tmaj_k": 1, "tmaj_stages": 3}, {"tmaj_tpc": 1}, {"tmaj_images": 1},
                                   {"tmaj_v8": 0}, {"pdl": 0}])
def test_convert_tma_kernel_variants(path, knobs):
    """The warp-specialised TMA kernels compiled per plan (default: 2-stage
    ring, 2 tiles per group and CTA) persistent (rings that wrap many
    times), one consumer group per CTA, one tile per CTA, no PDL, and the
    template kernels (tma_jit=0); configs 2 / 3 / 5 at small sizes, a ragged
    batch, and a CTA cap (many tiles per CTA)."""
    cases = [(configs.cfg2(batch_bits=0), 5, 0), (configs.cfg3(n_bits=9), 1, 3),
             (configs.cfg5(m_bits=9, kb_bits=9), 1, 2), (configs.cfg3(n_bits=9, m_bits=8), 2, 0)]
    for k, v in knobs.items():
        ll.tune(k, v)
    try:
        for c, batch, max_ctas in cases:
            w = c["elem_bytes"]
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            src = values_torch((1 << A.in_bits) * batch, 61, w, "cuda")
            dst = torch.zeros((1 << B.in_bits) * batch, dtype=src.dtype, device="cuda")
            ll.convert(src, A, dst, B, 8 * w, path=path, batch=batch, max_ctas=max_ctas)
            torch.cuda.synchronize()
            assert _np(dst, w).tobytes() == expect_convert(c, _np(src, w), batch).tobytes(), (path, knobs)
    finally:
        for k in knobs:
            ll.tune(k, {"tma_jit": 1, "pdl": 1, "tmaj_v8": 1}.get(k, 0))


@pytest.mark.parametrize("knobs", [{"ld_hint": 1}, {"ld_hint": 2}, {"ld_hint": 3}, {"st_hint": 1},
                                   {"st_hint": 2}, {"st_hint": 3}, {"st_hint": 4}, {"tile_order": 1},
                                   {"tile_order": 2}, {"tile_order": 12}, {"tile_order": 23},
                                   {"pdl_prefetch": 0}, {"pdl_prefetch": 2}, {"smem_jit_tpg": 0},
                                   {"tile_xor": 2}, {"tile_xor": 6}, {"tile_xor": 4, "tile_xor_skip": 0},
                                   {"pdl_prefetch_waves": 3}, {"pdl_prefetch_waves": 1}, {"pdl_prefetch_bulk": 0}])
def test_convert_smem_kernel_hint_and_order_knobs(knobs):
    """The compiled smem kernel under the cache-hint ablation (ld_hint /
    st_hint change only the global instructions' qualifiers) and the tile
    orders (a different tile -> CTA assignment): configs 2 / 3 / 5 at small
    sizes with a ragged batch and a CTA cap, byte-exact."""
    cases = [(configs.cfg2(batch_bits=0), 3, 0), (configs.cfg3(n_bits=9), 1, 3),
             (configs.cfg5(m_bits=9, kb_bits=9), 2, 0)]
    for k, v in knobs.items():
        ll.tune(k, v)
    try:
        for c, batch, max_ctas in cases:
            w = c["elem_bytes"]
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            assert ll.plan_describe(A, B, 8 * w)["path"] == "smem"
            src = values_torch((1 << A.in_bits) * batch, 67, w, "cuda")
            dst = torch.zeros((1 << B.in_bits) * batch, dtype=src.dtype, device="cuda")
            ll.convert(src, A, dst, B, 8 * w, batch=batch, max_ctas=max_ctas)
            torch.cuda.synchronize()
            assert _np(dst, w).tobytes() == expect_convert(c, _np(src, w), batch).tobytes(), knobs
    finally:
        for k in knobs:
            ll.tune(k, {"smem_jit_tpg": 1, "pdl_prefetch": 1, "tile_xor_skip": 1, "pdl_prefetch_waves": 2, "pdl_prefetch_bulk": 1}.get(k, 0))


def test_convert_shard_with_tile_xor():
    """The diagonal tile order (knob tile_xor) applies to full-range launches
    only: sharded conversions (ll_convert_shard) stay inside their slices."""
    c = configs.cfg5(m_bits=11, kb_bits=10)   # shardable (config 3 is not: a transpose)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    w = c["elem_bytes"]
    full = values_torch(1 << A.in_bits, 77, w, "cuda")
    exp = expect_convert(c, _np(full, w))
    ll.tune("tile_xor", 4)
    try:
        assert ll.plan_describe(A, B, 8 * w)["path"] == "smem"
        parts = []
        for r in range(4):
            s0, s1, d0, d1 = ll.shard_describe(A, B, 8 * w, 4, r)
            dl = torch.zeros(d1 - d0, dtype=torch.uint8, device="cuda")
            ll.convert_shard(full.view(torch.uint8)[s0:s1].clone(), A, dl, B, 8 * w, 4, r)
            torch.cuda.synchronize()
            parts.append((d0, dl.cpu().numpy().tobytes()))
        assert b"".join(b for _, b in sorted(parts)) == exp.tobytes()
    finally:
        ll.tune("tile_xor", 0)


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_register_permutation_prefetch(w):
    """The register-permutation kernel with the first wave's L2 prefetch
    before griddepcontrol.wait (knob regperm_prefetch, off by default),
    ragged batches, byte-exact."""
    rng = random.Random(1600 + w)
    ll.tune("regperm_prefetch", 1)
    try:
        for case in range(3):
            c = perm_pair(rng, rng.randint(12, 15), w, 2 + case % 2, "reg")
            batch = 1 + 2 * (case % 2)
            src, dst = run_convert(c, path="regperm", seed=case + 30, batch=batch)
            assert dst.tobytes() == expect_convert(c, src, batch).tobytes(), (w, case)
    finally:
        ll.tune("regperm_prefetch", 0)


@pytest.mark.parametrize("knobs", [{}, {"shuffle_pdl": 0}, {"pdl_prefetch": 0}, {"pdl_prefetch": 2},
                                   {"shuffle_prefetch_waves": 2}, {"shuffle_prefetch_waves": 1}, {"shuffle_prefetch_waves": 4},
                                   {"shuffle_prefetch_bulk": 0}])
def test_convert_shuffle_kernel_pdl(knobs):
    """The compiled HBM shuffle kernel launched with programmatic dependent
    launch (griddepcontrol.wait first) and the first wave's L2 prefetch:
    back-to-back launches where each reads what the previous one wrote
    (src -> tmp -> back), byte-exact; configs 6 and 2 at small sizes."""
    cases = [(configs.cfg6(n_bits=9, k_bits=9), 1), (configs.cfg2(batch_bits=2), 3)]
    for k, v in knobs.items():
        ll.tune(k, v)
    try:
        for c, batch in cases:
            w = c["elem_bytes"]
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            src = values_torch((1 << A.in_bits) * batch, 71, w, "cuda")
            mid = torch.zeros((1 << B.in_bits) * batch, dtype=src.dtype, device="cuda")
            back = torch.zeros_like(src)
            for _ in range(3):
                ll.convert(src, A, mid, B, 8 * w, path="shuffle", batch=batch)
                ll.convert(mid, B, back, A, 8 * w, path="shuffle", batch=batch)
            torch.cuda.synchronize()
            assert _np(mid, w).tobytes() == expect_convert(c, _np(src, w), batch).tobytes(), knobs
            assert _np(back, w).tobytes() == _np(src, w).tobytes(), knobs
    finally:
        for k in knobs:
            ll.tune(k, {"pdl_prefetch": 1, "shuffle_pdl": 1, "shuffle_prefetch_waves": 3, "shuffle_prefetch_bulk": 1}.get(k, 0))


@pytest.mark.parametrize("swz", [0, 1, 2, 3])
def test_convert_tma_each_swizzle_mode(swz):
    """Every hardware swizzle mode (the Def. 5 instances) executed on the
    device: the planner is pinned to one mode and must stay byte-exact."""
    ll.tune("tma_force_swizzle", swz)
    try:
        for c in (configs.cfg5(m_bits=9, kb_bits=9), configs.cfg3(n_bits=9),
                  configs.cfg2(batch_bits=2)):
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            try:
                plan = ll.plan_describe(A, B, 8 * c["elem_bytes"], "smem_tma")
            except ll.LLError:
                continue
            assert plan["tma"]["swizzle"] == ["none", "32B", "64B", "128B"][swz]
            src, dst = run_convert(c, path="smem_tma", seed=40 + swz)
            assert dst.tobytes() == expect_convert(c, src).tobytes()
    finally:
        ll.tune("tma_force_swizzle", -1)


@pytest.mark.parametrize("batch", [3, 37])
def test_convert_tma_ragged_batch(batch):
    c = configs.cfg2(batch_bits=0)
    src, dst = run_convert(c, path="smem_tma", batch=batch, seed=19)
    assert dst.tobytes() == expect_convert(c, src, batch).tobytes()


@pytest.mark.parametrize("batch", [3, 37])
def test_convert_shuffle_ragged_batch(batch):
    c = configs.cfg2(batch_bits=0)
    src, dst = run_convert(c, path="shuffle", batch=batch, seed=13)
    assert dst.tobytes() == expect_convert(c, src, batch).tobytes()


@pytest.mark.parametrize("name,mk,shards", [("cfg5", lambda: configs.cfg5(m_bits=10, kb_bits=8), 8),
                                            ("cfg2", lambda: configs.cfg2(batch_bits=3), 4),
                                            ("cfg2s", lambda: configs.cfg2(batch_bits=3), 2)])
@pytest.mark.parametrize("path", ["auto", "smem_tma", "smem_tma_store"])
def test_convert_shards_equal_full(name, mk, shards, path):
    """Each rank's shard converted from its own slices (separate allocations,
    SURVEY 8(e)) reassembles the oracle's full conversion."""
    c = mk()
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    src = values_torch(n, 29, w, "cuda")
    parts = []
    for r in range(shards):
        s0, s1, d0, d1 = ll.shard_describe(A, B, 8 * w, shards, r, path)
        sl = src.view(torch.uint8)[s0:s1].clone()          # this rank's memory only
        dl = torch.empty(d1 - d0, dtype=torch.uint8, device="cuda")
        ll.convert_shard(sl, A, dl, B, 8 * w, shards, r, path=path)
        parts.append(dl)
    torch.cuda.synchronize()
    got = torch.cat(parts).cpu().numpy().view(_NP[w])
    assert got.tobytes() == expect_convert(c, _np(src, w)).tobytes()


def test_convert_identity_is_copy():
    c = configs.cfg2(batch_bits=1)
    c = {"A": c["A"], "B": c["A"], "elem_bytes": 2}
    src, dst = run_convert(c)
    assert dst.tobytes() == src.tobytes()


def test_convert_roundtrip_on_device():
    c = configs.cfg5(m_bits=9, kb_bits=8)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    src = values_torch(1 << A.in_bits, 3, 1, "cuda")
    mid = torch.empty_like(src)
    back = torch.empty_like(src)
    ll.convert(src, A, mid, B, 8)
    ll.convert(mid, B, back, A, 8)
    torch.cuda.synchronize()
    assert torch.equal(src, back)


# ----------------------------------------------------------- full BASELINE sizes
#
# Whole destination buffers at the BASELINE sizes, element by element against
# the oracle (convert_np_chunks: the plain definition evaluated in chunks on
# the host), in the launch configuration bench.py times (AUTO) and on the TMA
# paths.  The expected buffer is computed once per config and compared on the
# device (torch.equal of the raw bits).

_FULL = {}
FULL_CONFIGS = {"cfg2": lambda: configs.cfg2(), "cfg3": lambda: configs.cfg3(),
                "cfg5": lambda: configs.cfg5(), "cfg2w": lambda: configs.cfg2w(),
                "cfg6": lambda: configs.cfg6()}


def full_expected(name):
    if name not in _FULL:
        _FULL.clear()       # keep one config's buffers resident at a time
        c = FULL_CONFIGS[name]()
        w = c["elem_bytes"]
        Ao, Bo = _olayout(c["A"]), _olayout(c["B"])
        src = values_torch(1 << Ao.in_bits, 17, w, "cuda")
        src_np = _np(src, w)
        exp = np.empty(1 << Bo.in_bits, dtype=_NP[w])
        for h0, d in oconv.convert_np_chunks(src_np, Ao, Bo):
            exp[h0:h0 + len(d)] = d
        exp_t = torch.from_numpy(exp.view({1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64}[w])).cuda()
        _FULL[name] = (c, src, exp_t)
    return _FULL[name]


@pytest.mark.parametrize("path", ["auto", "smem_tma", "smem_tma_store"])
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg5", "cfg6"])
def test_convert_full_size_whole_buffer(name, path):
    c, src, exp = full_expected(name)
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    dst = torch.empty_like(exp)
    ll.convert(src, A, dst, B, 8 * w, path=path)
    torch.cuda.synchronize()
    assert torch.equal(dst, exp), (name, path)


# ------------------------------------------------------------------------ gather

def run_gather(c, path, seed=4, batch=1):
    w = c["elem_bytes"]
    L = ll.Layout.from_spec(c["L"])
    n = (1 << L.in_bits) * batch
    src = values_torch(n, seed, w, "cuda")
    idx = indices_torch(n, seed + 1, c["idx_limit"], "cuda")
    out = torch.zeros_like(src)
    ll.gather(src, idx, out, L, c["axis"], 8 * w, path=path, batch=batch)
    torch.cuda.synchronize()
    return _np(src, w), idx.cpu().numpy(), _np(out, w)


@pytest.mark.parametrize("path", ["auto", "shuffle", "generic"])
@pytest.mark.parametrize("r_bits", [0, 3])
def test_gather_tile_axis(path, r_bits):
    c = configs.cfg4(r_bits=r_bits)
    src, idx, out = run_gather(c, path)
    exp = oconv.gather_np(src, idx, _olayout(c["L"]), c["axis"])
    assert out.tobytes() == exp.tobytes()


def test_gather_full_axis_direct():
    c = configs.cfg4(r_bits=2, variant="full")
    src, idx, out = run_gather(c, "auto")
    exp = oconv.gather_np(src, idx, _olayout(c["L"]), c["axis"])
    assert out.tobytes() == exp.tobytes()


@pytest.mark.parametrize("w", [1, 2, 8])
def test_gather_other_widths(w):
    c = configs.cfg4(r_bits=1)
    c = dict(c, elem_bytes=w)
    for path in ("shuffle", "generic"):
        src, idx, out = run_gather(c, path)
        exp = oconv.gather_np(src, idx, _olayout(c["L"]), c["axis"])
        assert out.tobytes() == exp.tobytes(), (w, path)


@pytest.mark.parametrize("u", [1, 4])
@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_gather_shuffle_vectors_in_flight(w, u):
    """Knob gather_shfl_u=u: the shuffle gather issues u warp-vectors'
    loads before the first shuffle; same bytes, including a ragged last
    iteration (warp-vectors not a multiple of u per grid stride)."""
    try:
        ll.tune("gather_shfl_u", u)
        for r_bits, batch in ((0, 1), (3, 3)):
            c = dict(configs.cfg4(r_bits=r_bits), elem_bytes=w)
            src, idx, out = run_gather(c, "shuffle", batch=batch)
            n = src.size // batch
            for k in range(batch):
                exp = oconv.gather_np(src[k * n:(k + 1) * n], idx[k * n:(k + 1) * n],
                                      _olayout(c["L"]), c["axis"])
                assert out[k * n:(k + 1) * n].tobytes() == exp.tobytes(), (w, r_bits, k)
    finally:
        ll.tune("gather_shfl_u", 2)


@pytest.mark.parametrize("variant", ["tile", "full"])
def test_gather_full_size_whole_buffer(variant):
    """Config 4 at the BASELINE size ([4096, 128, 32] fp32 tile axis, or the
    full 4096-long axis), whole output against the oracle (gather_np) and
    against torch.gather (a library routine on the row-major view)."""
    c = configs.cfg4(variant=variant)
    w = 4
    L = ll.Layout.from_spec(c["L"])
    n = 1 << L.in_bits
    src = values_torch(n, 4, w, "cuda")
    idx = indices_torch(n, 5, c["idx_limit"], "cuda")
    out = torch.empty_like(src)
    ll.gather(src, idx, out, L, c["axis"], 32)
    torch.cuda.synchronize()
    ref = torch.gather(src.view(-1, c["idx_limit"]), 1, idx.view(-1, c["idx_limit"]).long()).view(-1)
    assert torch.equal(ref, out)
    exp = oconv.gather_np(_np(src, w), idx.cpu().numpy(), _olayout(c["L"]), c["axis"])
    assert _np(out, w).tobytes() == exp.tobytes()


def rand_gather_layout(rng, w, n, a, region, mix):
    """A bijective distributed layout over n bits whose axis (the middle
    output dim, 2^a long) has all its preimage vectors L^{-1} e_axis inside
    the low `region` buffer bits; mix: random invertible column operations
    inside / outside the region (non-unit axis vectors, y_contig = 0)."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    x = rng.randint(1, 3)
    out = [("p", x), ("q", a), ("t", n - a - x)]
    flat_axis = [n - a - x + k for k in range(a)]          # bit positions of q in the flat index
    pos = rng.sample(range(region), a)
    cols = [None] * n
    for k, p_ in enumerate(pos):
        cols[p_] = 1 << flat_axis[k]
    rest = [b for b in range(n) if b not in flat_axis]
    rng.shuffle(rest)
    for p_ in range(n):
        if cols[p_] is None:
            cols[p_] = 1 << rest.pop()
    if mix:
        for _ in range(3 * n):
            i, j = rng.sample(range(n), 2)
            if (i < region) == (j < region):
                cols[i] ^= cols[j]
    r = rng.randint(max(0, vb - 1), vb + 2)
    nw = rng.randint(0, min(3, n - r - 5))
    dims = [("reg", r), ("lane", 5), ("warp", nw), ("block", n - r - 5 - nw)]
    tmp = OLayout([], out, {})
    bases, k = {}, 0
    for nm, b in dims:
        bases[nm] = [tmp.unflatten(c) for c in cols[k:k + b]]
        k += b
    return {"L": {"in_dims": dims, "out_dims": out, "bases": bases}, "axis": 1, "elem_bytes": w,
            "idx_limit": 1 << a}


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_gather_random_layouts_every_path(w):
    """P:719-727 on random distributed layouts with the axis bits placed
    anywhere inside a region (inside a warp's registers and lanes, inside a
    CTA unit, or anywhere), with unit and mixed (non-unit) axis vectors:
    every applicable path -- shuffle, smem, direct -- byte-exact against the
    oracle."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    rng = random.Random(900 + w)
    ran = {"shuffle": 0, "smem": 0, "generic": 0}
    for case in range(18):
        n = rng.randint(vb + 9, vb + 12)
        kind = case % 3
        region = [rng.randint(vb + 3, vb + 9), rng.randint(vb + 6, min(n, vb + 12)), n][kind]
        a = rng.randint(1, min(6, region))
        c = rand_gather_layout(rng, w, n, a, region, mix=case % 2 == 1)
        L = ll.Layout.from_spec(c["L"])
        for path in ("shuffle", "smem", "generic"):
            try:
                ll.gather_describe(L, 1, 8 * w, path)
            except ll.LLError:
                assert path != "generic"
                continue
            batch = 1 + case % 2 * 2
            src, idx, out = run_gather(c, path, seed=case * 7 + w, batch=batch)
            m = src.size // batch
            for b in range(batch):
                exp = oconv.gather_np(src[b * m:(b + 1) * m], idx[b * m:(b + 1) * m],
                                      _olayout(c["L"]), 1)
                assert out[b * m:(b + 1) * m].tobytes() == exp.tobytes(), (w, case, path, b)
            ran[path] += 1
    assert ran["shuffle"] >= 4 and ran["smem"] >= 6 and ran["generic"] == 18, ran


@pytest.mark.parametrize("path", ["shuffle", "smem"])
@pytest.mark.parametrize("variant", ["tile", "full"])
def test_gather_compiled_paths_configs(path, variant):
    """Config 4 (tile axis) and its full-axis variant at reduced rows on the
    compiled gather paths, where they apply (the full 4096 axis does not fit a
    warp: shuffle is rejected)."""
    c = configs.cfg4(r_bits=4, variant=variant)
    L = ll.Layout.from_spec(c["L"])
    try:
        ll.gather_describe(L, c["axis"], 32, path)
    except ll.LLError:
        assert (path, variant) == ("shuffle", "full")
        return
    src, idx, out = run_gather(c, path)
    exp = oconv.gather_np(src, idx, _olayout(c["L"]), c["axis"])
    assert out.tobytes() == exp.tobytes()


@pytest.mark.parametrize("path,knobs", [("smem", {"gather_smem_upc": 0}), ("smem", {"gather_smem_upc": 3}),
                                         ("shuffle", {"gather_shfl_waves": 8}), ("shuffle", {"gather_shfl_waves": 1}),
                                         ("smem", {"gather_prefetch_waves": 0}), ("smem", {"gather_prefetch_waves": 4}),
                                         ("smem", {"gather_prefetch_waves": 2, "gather_smem_upc": 0})])
def test_gather_launch_shapes(path, knobs):
    """The compiled gathers' launch shapes (one pass by default; persistent /
    several units per CTA / grid-stride) on config 4 and its full-axis
    variant, byte-exact."""
    defaults = {"gather_smem_upc": 1, "gather_shfl_waves": -1, "gather_prefetch_waves": 1}
    for k, v in knobs.items():
        ll.tune(k, v)
    try:
        for variant in ("tile", "full"):
            c = configs.cfg4(r_bits=5, variant=variant)
            L = ll.Layout.from_spec(c["L"])
            try:
                ll.gather_describe(L, c["axis"], 32, path)
            except ll.LLError:
                continue
            src, idx, out = run_gather(c, path)
            exp = oconv.gather_np(src, idx, _olayout(c["L"]), c["axis"])
            assert out.tobytes() == exp.tobytes(), (path, knobs, variant)
    finally:
        for k in knobs:
            ll.tune(k, defaults[k])


@pytest.mark.parametrize("path", ["shuffle", "smem"])
@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_gather_timed_one_cta(path, w):
    """ll_gather_timed (the one-CTA in-kernel study): the first unit of the
    output equals the oracle's gather after `reps` repeated exchanges, and the
    cycle count is positive."""
    c = dict(configs.cfg4(r_bits=3), elem_bytes=w)
    L = ll.Layout.from_spec(c["L"])
    d = ll.gather_describe(L, c["axis"], 8 * w, path)
    ub = d["warp_unit_bits"] if path == "shuffle" else d["cta_unit_bits"]
    n = 1 << L.in_bits
    src = values_torch(n, 31, w, "cuda")
    idx = indices_torch(n, 32, 32, "cuda")
    out = torch.zeros_like(src)
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    ll.gather_timed(src, idx, out, L, c["axis"], 8 * w, path, 5, cyc)
    torch.cuda.synchronize()
    exp = oconv.gather_np(_np(src, w), idx.cpu().numpy(), _olayout(c["L"]), c["axis"])
    assert _np(out, w)[:1 << ub].tobytes() == exp[:1 << ub].tobytes()
    assert int(cyc.item()) > 0


def test_gather_out_of_range_check(monkeypatch):
    monkeypatch.setenv("LL_GATHER_CHECK", "1")
    c = configs.cfg4(r_bits=0)
    L = ll.Layout.from_spec(c["L"])
    n = 1 << L.in_bits
    src = values_torch(n, 1, 4, "cuda")
    idx = torch.zeros(n, dtype=torch.int32, device="cuda")
    idx[100] = 40
    out = torch.empty_like(src)
    with pytest.raises(ll.LLError) as e:
        ll.gather(src, idx, out, L, 2, 32)
    assert e.value.name == "LL_ERR_RANGE"


def test_convert_host_e2e():
    c = configs.cfg2(batch_bits=0)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    batch = 9
    n = (1 << 14) * batch
    src_h = values_torch(n, 21, 2, "cpu").pin_memory()
    dst_h = torch.empty_like(src_h).pin_memory()
    scratch = 4 * (1 << 15)
    ds = torch.empty(scratch // 2, dtype=torch.int16, device="cuda")
    dd = torch.empty(scratch // 2, dtype=torch.int16, device="cuda")
    ll.convert_host(src_h, A, dst_h, B, 16, batch, ds, dd, scratch)
    exp = expect_convert(c, src_h.numpy().view(np.uint16), batch)
    assert dst_h.numpy().view(np.uint16).tobytes() == exp.tobytes()


def test_misaligned_pointer_rejected():
    c = configs.cfg2(batch_bits=0)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    buf = torch.zeros((1 << 14) + 8, dtype=torch.int16, device="cuda")
    with pytest.raises(ll.LLError) as e:
        ll.convert(buf[1:], A, buf, B, 16)
    assert e.value.name == "LL_ERR_ARG"


# ------------------------------------------------------------ broadcast layouts

def _bcast_pair(rng, d, w, zeros_a, zeros_b, low_ok=False):
    """Distributed layouts over a d-bit tensor with zero columns (broadcast,
    P:528-537): zeros_a / zeros_b extra warp/block bits of A / B map to 0
    (replicated warps / blocks), or anywhere when low_ok."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    out = [("i", d // 2), ("j", d - d // 2)]
    tmp = OLayout([], out, {})
    specs = []
    for z in (zeros_a, zeros_b):
        n = d + z
        names = [("reg", vb + 1), ("lane", 5)]
        rest = n - vb - 1 - 5
        nw = min(rest, 2)
        names += [("warp", nw), ("block", rest - nw)]
        cols = [1 << k for k in range(d)]
        rng.shuffle(cols)
        if low_ok:
            allc = cols + [0] * z
            rng.shuffle(allc)
        else:
            # zeros in the high (warp / block) positions only
            head = cols[:vb + 1 + 5]
            tail = cols[vb + 1 + 5:] + [0] * z
            rng.shuffle(tail)
            allc = head + tail
        bases, k = {}, 0
        for nme, b in names:
            bases[nme] = [tmp.unflatten(x) for x in allc[k:k + b]]
            k += b
        specs.append({"in_dims": names, "out_dims": out, "bases": bases})
    return {"A": specs[0], "B": specs[1], "elem_bytes": w}


@pytest.mark.parametrize("w", [1, 2, 4])
@pytest.mark.parametrize("za,zb,low", [(0, 2, False), (2, 0, False), (1, 1, False), (2, 2, True)])
def test_convert_broadcast_layouts(w, za, zb, low):
    """Zero columns in B (destination copies, every copy written) and in A
    (source copies, the lowest preimage is read).  High zero
    columns stay on the tiled smem path; low ones fall back to the generic
    kernel."""
    rng = random.Random(700 + 10 * w + za + 3 * zb + (100 if low else 0))
    for _ in range(4):
        c = _bcast_pair(rng, rng.randint(12, 14), w, za, zb, low)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        path = ll.plan_describe(A, B, 8 * w)["path"]
        if not low:
            assert path in ("smem", "shuffle"), path
        src, dst = run_convert(c, seed=rng.randint(0, 999))
        assert dst.tobytes() == expect_convert(c, src).tobytes()


def reg_bcast_pair(rng, d, w, za, zb):
    """Distributed layouts over a d-bit tensor whose REGISTER bits carry
    zero columns ("registers 4-7 map to the same tensor elements
    as registers 0-3"): za / zb zero columns placed among A's / B's register
    bits, inside or above the 16-byte vector."""
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    out = [("i", d // 2), ("j", d - d // 2)]
    tmp = OLayout([], out, {})
    specs = []
    for z in (za, zb):
        r = vb + 1 + z
        n = d + z
        rest = n - r - 5
        nw = min(rest, 2)
        names = [("reg", r), ("lane", 5), ("warp", nw), ("block", rest - nw)]
        cols = [1 << k for k in range(d)]
        rng.shuffle(cols)
        regc = cols[:vb + 1] + [0] * z
        rng.shuffle(regc)
        allc = regc + cols[vb + 1:]
        bases, k = {}, 0
        for nme, b in names:
            bases[nme] = [tmp.unflatten(x) for x in allc[k:k + b]]
            k += b
        specs.append({"in_dims": names, "out_dims": out, "bases": bases})
    return {"A": specs[0], "B": specs[1], "elem_bytes": w}


@pytest.mark.parametrize("w", [1, 2, 4, 8])
@pytest.mark.parametrize("za,zb", [(1, 0), (0, 1), (1, 1), (2, 0), (0, 2), (2, 1)])
def test_convert_register_broadcast(w, za, zb):
    """Zero columns in register bits stay on the swizzled smem path (broadcast
    dedup): each distinct element crosses shared memory once;
    source copies are dropped after the load, destination copies are made in
    registers or by extra stores.  Byte-exact against the oracle (lowest
    preimage), and equal to the naive plan (knob bcast_dedup=0)."""
    rng = random.Random(1300 + 17 * w + 5 * za + zb)
    dedup = 0
    for _ in range(5):
        c = reg_bcast_pair(rng, rng.randint(12, 15), w, za, zb)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        seed = rng.randint(0, 999)
        src, dst = run_convert(c, seed=seed)           # AUTO (cost model: dedup or generic)
        exp = expect_convert(c, src).tobytes()
        assert dst.tobytes() == exp
        try:
            d = ll.plan_describe(A, B, 8 * w, "smem")
        except ll.LLError:
            d = {}
        if "bcast_dedup" in d:
            dedup += 1
            _, dsm = run_convert(c, path="smem", seed=seed)
            assert dsm.tobytes() == exp
        ll.tune("bcast_dedup", 0)
        try:
            _, dst0 = run_convert(c, seed=seed)
        finally:
            ll.tune("bcast_dedup", 1)
        assert dst0.tobytes() == exp
    assert dedup >= (3 if w > 1 else 2), dedup


@pytest.mark.parametrize("fam", ["blocked", "mma"])
def test_convert_sliced_layouts(fam):
    """Sliced layouts from blocked / mma parents over [512, 32]
    (4 warps, 8 CTAs), sliced along dim 1 with ll_slice: sliced<blocked> ->
    sliced<mma> and back, batched, byte-exact; the broadcast-dedup smem plan."""
    from oracle import shapeops
    from workloads.configs import spec as mkspec
    out = [("i", 9), ("j", 5)]
    pb = OLayout(**mkspec([("reg", ["j0", "j1", "j2", "i0"]), ("lane", ["j3", "j4", "i1", "i2", "i3"]),
                           ("warp", ["i4", "i5"]), ("block", ["i6", "i7", "i8"])], out))
    pm = OLayout(**mkspec([("reg", ["j0", "i3", "j3", "j4"]), ("lane", ["j1", "j2", "i0", "i1", "i2"]),
                           ("warp", ["i4", "i5"]), ("block", ["i6", "i7", "i8"])], out))

    def to_spec(L):
        return {"in_dims": L.in_dims, "out_dims": L.out_dims, "bases": {k: list(v) for k, v in L.bases.items()}}
    sb, sm = shapeops.slice_(pb, 1), shapeops.slice_(pm, 1)
    # the ABI's ll_slice agrees with the oracle's
    for par, sl in ((pb, sb), (pm, sm)):
        got = ll.slice_layout(ll.Layout.from_spec(to_spec(par)), 1).spec()["bases"]
        assert got == {k: [tuple(x) for x in v] for k, v in to_spec(sl)["bases"].items()}
    A, B = (sb, sm) if fam == "blocked" else (sm, sb)
    c = {"A": to_spec(A), "B": to_spec(B), "elem_bytes": 2}
    d = ll.plan_describe(ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"]), 16, "smem")
    assert d["path"] == "smem" and "bcast_dedup" in d, d["path"]
    for path in ("smem", "auto"):
        src, dst = run_convert(c, path=path, batch=64, seed=5)
        assert dst.tobytes() == expect_convert(c, src, 64).tobytes(), path


@pytest.mark.parametrize("mb,nb", [(6, 6), (7, 9), (10, 8)])
def test_fp8_transpose_paths(mb, nb):
    """fig:matrix-size workload: fp8 transposes through the three
    staging layouts agree with the oracle."""
    c = configs.cfg3(n_bits=nb, m_bits=mb)
    c = dict(c, elem_bytes=1)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    for path in ("smem", "smem_padded", "smem_noswizzle", "smem_tma"):
        if path == "smem_tma":
            try:   # fp8 transposes need 16x16 elements (256 B) per reader thread
                ll.plan_describe(A, B, 8, path)
            except ll.LLError:
                continue
        src, dst = run_convert(c, path=path, seed=mb * 31 + nb)
        assert dst.tobytes() == expect_convert(c, src).tobytes(), path


# ------------------------------------------------------------- mxfp4 upcast

@pytest.mark.parametrize("mb,kb,dist", [(8, 7, "narrow"), (9, 9, "narrow"), (9, 8, "uniform"),
                                        (8, 8, "edges")])
def test_mxfp4_upcast(mb, kb, dist):
    """NEXT #1: config-5 layouts, E2M1 bytes + E8M0 scales, bit-exact
    bf16.  narrow: scales in [120, 135] plus edge scales (0, 1, 254, 255 = NaN);
    uniform: every scale byte 0..255 (vectors mix the kernel's normal-product
    fast path with its general path); edges: only 0-3 and 251-255 (the fast
    path's bounds 2 and 252, subnormal and infinite products)."""
    from oracle import mxfp4
    c = configs.cfg5(m_bits=mb, kb_bits=kb)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    packed = values_torch(n, 41, 1, "cuda")
    n_sc = (1 << mb) * (1 << (kb - 4))
    if dist == "narrow":
        sc = (indices_torch(n_sc, 42, 16, "cuda") + 120).to(torch.uint8)
        sc[:4] = torch.tensor([0, 1, 254, 255], dtype=torch.uint8)
    elif dist == "uniform":
        sc = indices_torch(n_sc, 43, 256, "cuda").to(torch.uint8)
    else:
        pick = torch.tensor([0, 1, 2, 3, 251, 252, 253, 254, 255], dtype=torch.uint8, device="cuda")
        sc = pick[indices_torch(n_sc, 44, 9, "cuda").long()]
    out = torch.empty(2 * n, dtype=torch.int16, device="cuda")
    ll.mxfp4_upcast(packed, A, sc, out, B)
    torch.cuda.synchronize()
    exp = mxfp4.upcast_np(_np(packed, 1), _olayout(c["A"]), sc.cpu().numpy(), _olayout(c["B"]))
    assert out.cpu().numpy().view(np.uint16).tobytes() == exp.tobytes()


@pytest.mark.parametrize("jit", [0, 1])
@pytest.mark.parametrize("dist", ["narrow", "uniform", "edges"])
def test_mxfp4_upcast_kernels(dist, jit):
    """Both upcast executors -- the template kernel and the one compiled for
    the plan (knob upcast_jit) -- bit-exact on every scale distribution."""
    ll.tune("upcast_jit", jit)
    try:
        test_mxfp4_upcast(9, 8, dist)
    finally:
        ll.tune("upcast_jit", 1)


@pytest.mark.parametrize("pdl", [0, 1])
def test_mxfp4_upcast_pdl_back_to_back(pdl):
    """The compiled upcast with and without programmatic dependent launch
    (knob upcast_pdl), three rounds of input generation + upcast back to back
    (each launch follows the kernels that wrote its inputs): bit-exact every
    time."""
    ll.tune("upcast_pdl", pdl)
    try:
        for _ in range(3):
            test_mxfp4_upcast(9, 8, "uniform")
    finally:
        ll.tune("upcast_pdl", 0)


@pytest.mark.parametrize("dist", ["narrow", "uniform"])
def test_mxfp4_upcast_full_size_whole_buffer(dist):
    """Config 5 at the BASELINE size (packed [32768, 16384] u8 -> 2 GiB of
    bf16), the launch bench.py --upcast times; the whole destination against
    the oracle (upcast_np_chunks: A's preimage, OCP MX table), chunk by chunk
    on the device."""
    from oracle import mxfp4
    c = configs.cfg5()
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    packed = values_torch(n, 51, 1, "cuda")
    n_sc = n // 16
    if dist == "narrow":
        sc = (indices_torch(n_sc, 52, 16, "cuda") + 120).to(torch.uint8)
    else:
        sc = indices_torch(n_sc, 53, 256, "cuda").to(torch.uint8)
    out = torch.empty(2 * n, dtype=torch.int16, device="cuda")
    ll.mxfp4_upcast(packed, A, sc, out, B)
    torch.cuda.synchronize()
    for h0, exp in mxfp4.upcast_np_chunks(_np(packed, 1), _olayout(c["A"]), sc.cpu().numpy(),
                                          _olayout(c["B"]), chunk=1 << 24):
        e = torch.from_numpy(exp.view(np.int16)).cuda()
        assert torch.equal(out[2 * h0:2 * h0 + e.numel()], e), h0


# ------------------------------------------------------------- checksum (a12)

@pytest.mark.parametrize("w", [1, 2, 4, 8])
@pytest.mark.parametrize("n,base", [(0, 0), (1, 0), (37, 5), (4099, 0), (1 << 20, 123456789)])
def test_checksum_matches_oracle(w, n, base):
    from oracle import checksum as ock
    buf = values_torch(max(n, 1), 61 + w, w, "cuda")
    res = torch.zeros(1, dtype=torch.int64, device="cuda")
    for indexed in (True, False):
        ll.checksum(buf, n, 8 * w, res, indexed=indexed, index_base=base)
        torch.cuda.synchronize()
        got = int(res.item()) & ((1 << 64) - 1)
        assert got == ock.checksum_np(_np(buf, w)[:n], indexed=indexed, base=base)


def test_checksum_full_size_conversion_properties():
    """cfg5 at full size: the index-free checksum of dst equals src's (the
    conversion is a permutation); per-shard indexed checksums (each with its
    slice's base) add up to the whole destination's."""
    c = configs.cfg5()
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    src = values_torch(n, 71, 1, "cuda")
    dst = torch.empty_like(src)
    ll.convert(src, A, dst, B, 8)
    res = torch.zeros(4, dtype=torch.int64, device="cuda")
    ll.checksum(src, n, 8, res[0:1], indexed=False)
    ll.checksum(dst, n, 8, res[1:2], indexed=False)
    ll.checksum(dst, n, 8, res[2:3], indexed=True)
    parts = 0
    for k in range(8):
        s0, s1, d0, d1 = ll.shard_describe(A, B, 8, 8, k)
        ll.checksum(dst[d0:], d1 - d0, 8, res[3:4], indexed=True, index_base=d0)
        torch.cuda.synchronize()
        parts = (parts + int(res[3].item())) & ((1 << 64) - 1)
    torch.cuda.synchronize()
    r = [int(x) & ((1 << 64) - 1) for x in res.cpu().tolist()]
    assert r[0] == r[1]
    assert parts == r[2]


@pytest.mark.parametrize("ramp,chunk_mb", [(2, 32), (0, 32), (2, 1), (4, 1), (3, 2)])
def test_convert_host_sharded_single_instance(ramp, chunk_mb):
    """One large instance (8 MiB) chunked by shards through ll_convert_host,
    uniform chunks (host_ramp 0) or a ramped schedule whose first and last
    chunks are cut into 1/2^R .. 1/2 pieces, 1-32 MiB chunks."""
    c = configs.cfg5(m_bits=12, kb_bits=11)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    src_h = values_torch(n, 23, 1, "cpu").pin_memory()
    dst_h = torch.empty_like(src_h).pin_memory()
    scratch = 4 << 20
    ds = torch.empty(scratch, dtype=torch.uint8, device="cuda")
    dd = torch.empty(scratch, dtype=torch.uint8, device="cuda")
    ll.tune("host_ramp", ramp)
    ll.tune("host_chunk_mb", chunk_mb)
    try:
        ll.convert_host(src_h, A, dst_h, B, 8, 1, ds, dd, scratch)
    finally:
        ll.tune("host_ramp", 0)
        ll.tune("host_chunk_mb", 0)
    exp = expect_convert(c, src_h.numpy())
    assert dst_h.numpy().tobytes() == exp.tobytes()


@pytest.mark.parametrize("n_shards,chunk_mb", [(2, 1), (4, 32), (8, 1)])
def test_convert_host_shard(n_shards, chunk_mb):
    """ll_convert_host_shard: every rank's shard from its host slices, cut
    into sub-shards and pipelined; the slices reassemble to the oracle's
    whole destination (config 5 family, 8 MiB)."""
    c = configs.cfg5(m_bits=12, kb_bits=11)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    src = values_torch(n, 29, 1, "cpu")
    exp = expect_convert(c, src.numpy())
    scratch = 2 << 20
    ds = torch.empty(scratch, dtype=torch.uint8, device="cuda")
    dd = torch.empty(scratch, dtype=torch.uint8, device="cuda")
    ll.tune("host_chunk_mb", chunk_mb)
    try:
        parts = []
        for r in range(n_shards):
            s0, s1, d0, d1 = ll.shard_describe(A, B, 8, n_shards, r)
            src_h = src[s0:s1].clone().pin_memory()
            dst_h = torch.zeros(d1 - d0, dtype=torch.uint8).pin_memory()
            ll.convert_host_shard(src_h, A, dst_h, B, 8, n_shards, r, ds, dd, scratch)
            parts.append((d0, dst_h.numpy().tobytes()))
    finally:
        ll.tune("host_chunk_mb", 0)
    assert b"".join(b for _, b in sorted(parts)) == exp.tobytes()


@pytest.mark.parametrize("host_2d", [1, 0])
def test_convert_host_pitched_transpose(host_2d):
    """A single 8 MiB transpose through ll_convert_host with 1 MiB chunks:
    pitched shards (contiguous dst slices, 1 KiB src rows; host_2d=1) or the
    whole instance at once (host_2d=0), both byte-exact."""
    c = configs.cfg3(n_bits=11)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    src_h = values_torch(n, 31, 2, "cpu").pin_memory()
    dst_h = torch.zeros_like(src_h).pin_memory()
    ds = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    dd = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    try:
        ll.tune("host_chunk_mb", 1)
        ll.tune("host_2d", host_2d)
        ll.convert_host(src_h, A, dst_h, B, 16, 1, ds, dd, 2 * n)
    finally:
        ll.tune("host_chunk_mb", 0)
        ll.tune("host_2d", 1)
    exp = expect_convert(c, _np(src_h, 2))
    assert _np(dst_h, 2).tobytes() == exp.tobytes()


def test_gather_host_e2e():
    """ll_gather_host: 300 [128, 32] instances (4.7 MiB of values) from pinned
    host buffers in 1 MiB chunks (a ragged last chunk), byte-exact per
    instance against the oracle."""
    c = configs.cfg4(r_bits=0)
    L = ll.Layout.from_spec(c["L"])
    m = 1 << L.in_bits
    batch = 300
    src_h = values_torch(m * batch, 41, 4, "cpu").pin_memory()
    idx_h = indices_torch(m * batch, 42, c["idx_limit"], "cpu").pin_memory()
    out_h = torch.zeros_like(src_h).pin_memory()
    scratch = 2 << 20
    bufs = [torch.empty(scratch, dtype=torch.uint8, device="cuda") for _ in range(3)]
    try:
        ll.tune("host_chunk_mb", 1)
        ll.gather_host(src_h, idx_h, out_h, L, c["axis"], 32, batch, *bufs, scratch)
    finally:
        ll.tune("host_chunk_mb", 0)
    src, idx, out = _np(src_h, 4), idx_h.numpy(), _np(out_h, 4)
    for b in range(batch):
        exp = oconv.gather_np(src[b * m:(b + 1) * m], idx[b * m:(b + 1) * m], _olayout(c["L"]), c["axis"])
        assert out[b * m:(b + 1) * m].tobytes() == exp.tobytes(), b


# ------------------------------------------------ register-faithful path (regs)

def rand_faithful_pair(rng, w, match_lanes):
    """A: random bit-permutation layout (reg, lane, warp, block); B: the same
    block columns, its (reg, lane, warp) a random permutation of A's; with
    match_lanes B keeps A's lanes 0, 1 (ldmatrix / stmatrix both apply)."""
    kw = {1: 2, 2: 1, 4: 0}[w]
    r = rng.randint(max(kw, 1), 6)
    nw = rng.randint(0, 3)
    nb = rng.randint(0, 3)
    d = r + 5 + nw
    tot = d + nb
    out = [("i", tot // 2), ("j", tot - tot // 2)]
    tmp = OLayout([], out, {})
    cols = [1 << k for k in range(tot)]
    rng.shuffle(cols)
    tile, blk = cols[:d], cols[d:]
    perm = tile[:]
    while True:
        rng.shuffle(perm)
        if match_lanes:
            a0, a1 = tile[r], tile[r + 1]
            perm.remove(a0)
            perm.remove(a1)
            perm[r:r] = [a0, a1]
        # B's word must hold elements A holds in registers (prmt on load)
        if all(x in tile[:r] for x in perm[:kw]):
            break
        perm = tile[:]
    names = [("reg", r), ("lane", 5), ("warp", nw), ("block", nb)]

    def spec(v):
        bases, k = {}, 0
        for n, b in names:
            bases[n] = [tmp.unflatten(x) for x in v[k:k + b]]
            k += b
        return {"in_dims": names, "out_dims": out, "bases": bases}
    return {"A": spec(tile + blk), "B": spec(perm + blk), "elem_bytes": w}


@pytest.mark.parametrize("mat", [1, 0])
@pytest.mark.parametrize("name,mk", [("cfg1a", lambda: configs.cfg1("mma")),
                                     ("cfg1b", lambda: configs.cfg1("T")),
                                     ("cfg2_b3", lambda: configs.cfg2(batch_bits=3))])
def test_convert_regs_configs(name, mk, mat):
    """Register-faithful execution of configs 1-2 (threads = the layouts' own
    lanes and warps), with stmatrix / ldmatrix allowed or not."""
    c = mk()
    ll.tune("regs_matrix", mat)
    try:
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        plan = ll.plan_describe(A, B, 8 * c["elem_bytes"], "regs")
        if name == "cfg1a":
            assert (plan["regs"]["write"] == "stmatrix") == bool(mat)
        src, dst = run_convert(c, path="regs")
        assert dst.tobytes() == expect_convert(c, src).tobytes(), plan["regs"]
    finally:
        ll.tune("regs_matrix", 1)


@pytest.mark.parametrize("w", [1, 2, 4])
@pytest.mark.parametrize("match_lanes", [False, True])
def test_convert_regs_random_pairs(w, match_lanes):
    rng = random.Random(800 + 10 * w + match_lanes)
    kinds = set()
    for _ in range(12):
        c = rand_faithful_pair(rng, w, match_lanes)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        plan = ll.plan_describe(A, B, 8 * w, "regs")
        if "regs" in plan:       # (else the cost model chose the shuffle exchange)
            kinds.add((plan["regs"]["write"], plan["regs"]["read"]))
        batch = rng.choice([1, 3])
        src, dst = run_convert(c, path="regs", seed=rng.randint(0, 999), batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes(), plan.get("regs")
    if match_lanes:
        assert ("stmatrix", "ldmatrix") in kinds


def test_convert_regs_timed_cycles():
    """In-kernel repetition (reps) leaves the result unchanged and reports
    per-CTA cycles that grow with reps."""
    c = configs.cfg1("mma")
    w = 2
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    src = values_torch(1 << A.in_bits, 9, w, "cuda")
    exp = expect_convert(c, _np(src, w))
    cyc = []
    for reps in (1, 1, 256):      # the first launch warms the instruction cache
        dst = torch.zeros_like(src)
        cy = torch.zeros(4, dtype=torch.int64, device="cuda")
        ll.convert_regs_timed(src, A, dst, B, 16, reps=reps, cycles=cy)
        torch.cuda.synchronize()
        assert _np(dst, w).tobytes() == exp.tobytes()
        cyc.append(int(cy[0].item()))
    assert 0 < cyc[1] < cyc[2]


def rand_warp_local_pair(rng, w):
    """Random reg/lane/warp/block pair whose exchange stays inside each warp:
    B keeps A's warp and block columns and permutes A's (reg, lane) ones."""
    kw = {1: 2, 2: 1, 4: 0}[w]
    r = rng.randint(max(kw, 1), 5)
    nw = rng.randint(0, 2)
    nb = rng.randint(0, 2)
    d = r + 5 + nw
    tot = d + nb
    out = [("i", tot // 2), ("j", tot - tot // 2)]
    tmp = OLayout([], out, {})
    cols = [1 << k for k in range(tot)]
    rng.shuffle(cols)
    rl, rest = cols[:r + 5], cols[r + 5:]
    while True:
        perm = rl[:]
        rng.shuffle(perm)
        if all(x in rl[:r] for x in perm[:kw]):
            break
    names = [("reg", r), ("lane", 5), ("warp", nw), ("block", nb)]

    def spec(v):
        bases, k = {}, 0
        for n, b in names:
            bases[n] = [tmp.unflatten(x) for x in v[k:k + b]]
            k += b
        return {"in_dims": names, "out_dims": out, "bases": bases}
    return {"A": spec(rl + rest), "B": spec(perm + rest), "elem_bytes": w}


def test_convert_regs_shuffle_cfg2w():
    """The paper's warp-shuffle exchange, register-faithful, in the
    NVRTC-specialised kernel: warp-aligned config-2 pair, batch of tiles."""
    c = configs.cfg2w(batch_bits=4)
    src, dst = run_convert(c, path="regs_shuffle", seed=21)
    assert dst.tobytes() == expect_convert(c, src).tobytes()


@pytest.mark.parametrize("w", [1, 2, 4])
def test_convert_regs_shuffle_random_pairs(w):
    rng = random.Random(1000 + w)
    done = 0
    for _ in range(40):
        if done == 6:
            break
        c = rand_warp_local_pair(rng, w)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            ll.plan_describe(A, B, 8 * w, "regs_shuffle")
        except ll.LLError:
            continue
        batch = rng.choice([1, 3])
        src, dst = run_convert(c, path="regs_shuffle", seed=rng.randint(0, 999), batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes()
        done += 1
    assert done >= 3


def test_regs_shuffle_timed_round_trips():
    """reps A -> B -> A round trips inside the kernel leave the final A -> B
    result exact, and the cycles grow with reps."""
    c = configs.cfg2w(batch_bits=0)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    src = values_torch(1 << A.in_bits, 5, 2, "cuda")
    exp = expect_convert(c, _np(src, 2))
    cyc = []
    for reps in (1, 1, 64):       # the first launch warms the instruction cache
        dst = torch.zeros_like(src)
        cy = torch.zeros(4, dtype=torch.int64, device="cuda")
        ll.convert_regs_timed(src, A, dst, B, 16, reps=reps, cycles=cy, path="regs_shuffle")
        torch.cuda.synchronize()
        assert _np(dst, 2).tobytes() == exp.tobytes()
        cyc.append(int(cy[0].item()))
    assert 0 < cyc[1] < cyc[2]


def test_regs_register_permutation_and_cost_model():
    """Identical lanes and warps: the exchange is a register permutation
    inside each thread -- no shuffle in the generated kernel --
    and the regs path's cost model takes it; byte-exact."""
    rng = random.Random(77)
    c = rand_warp_local_pair(rng, 2)
    # keep A's lanes in B: permute only the register columns
    B = {k: (dict(v) if isinstance(v, dict) else v) for k, v in c["A"].items()}
    regs = list(B["bases"]["reg"])
    rng.shuffle(regs)
    B["bases"] = dict(B["bases"], reg=regs)
    c = dict(c, B=B)
    A_, B_ = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    plan = ll.plan_describe(A_, B_, 16, "regs")
    assert plan["path"] == "regs_shuffle"
    assert plan["regs_shuffle"]["exchange"] == "register permutation"
    assert "__shfl_sync" not in ll.jit_source(A_, B_, 16)
    src, dst = run_convert(c, path="regs", seed=8, batch=2)
    assert dst.tobytes() == expect_convert(c, src, 2).tobytes()


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_tiny_layouts(w):
    """Degenerate sizes: 1 to 64 elements (less than one 16-byte vector, less
    than a warp), a layout with no input bits at all, and the identity; every
    AUTO plan (copy / generic) stays byte-exact."""
    rng = random.Random(1100 + w)
    for d in range(0, 7):
        out = [("i", d // 2), ("j", d - d // 2)]
        for _ in range(3):
            dims = [("reg", rng.randint(0, d))]
            dims.append(("lane", d - dims[0][1]))
            specs = []
            for _k in range(2):
                cols = [1 << k for k in range(d)]
                rng.shuffle(cols)
                tmp = OLayout([], out, {})
                bases, k = {}, 0
                for n, b in dims:
                    bases[n] = [tmp.unflatten(x) for x in cols[k:k + b]]
                    k += b
                specs.append({"in_dims": dims, "out_dims": out, "bases": bases})
            c = {"A": specs[0], "B": specs[1], "elem_bytes": w}
            src, dst = run_convert(c, seed=d + 17)
            assert dst.tobytes() == expect_convert(c, src).tobytes(), (d, dims)


@pytest.mark.parametrize("name,path", [("cfg2", "regs"), ("cfg2w", "regs_shuffle")])
def test_convert_regs_full_size_whole_buffer(name, path):
    """Register-faithful paths at the BASELINE size (4096 tiles of 128x128
    fp16): the whole destination against the oracle."""
    c, src, exp = full_expected(name)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    dst = torch.empty_like(exp)
    ll.convert(src, A, dst, B, 16, path=path)
    torch.cuda.synchronize()
    assert torch.equal(dst, exp), (name, path)


@pytest.mark.parametrize("w", [1, 2, 4, 8])
def test_convert_smem_generic_kernel(w):
    """The generic (uncompiled) shared-memory kernel (knob smem_jit=0; the
    default compiles the plan, covered by every other smem test): configs and
    random pairs byte-exact against the oracle."""
    rng = random.Random(1200 + w)
    ll.tune("smem_jit", 0)
    try:
        cases = [rand_pair(rng, rng.randint(12, 16), w) for _ in range(8)]
        if w == 2:
            cases += [configs.cfg2(batch_bits=2), configs.cfg3(n_bits=9)]
        if w == 1:
            cases += [configs.cfg5(m_bits=9, kb_bits=8)]
        for c in cases:
            batch = rng.choice([1, 3])
            src, dst = run_convert(c, path="smem", seed=rng.randint(0, 999), batch=batch)
            assert dst.tobytes() == expect_convert(c, src, batch).tobytes()
    finally:
        ll.tune("smem_jit", 1)


def rand_trans_pair(rng, r):
    """A random reg/lane/warp/block fp16 layout and its "transpose" partner:
    B's word and lanes 0, 1 are A's lanes 2..4 and B's lanes 2..4 are A's word
    and lanes 0, 1 (an mma fragment and the fragment of the transposed tile):
    the pair the ldmatrix / stmatrix .trans tile lowers."""
    nw, nb = rng.randint(0, 2), rng.randint(0, 2)
    tot = r + 5 + nw + nb
    out = [("i", tot // 2), ("j", tot - tot // 2)]
    tmp = OLayout([], out, {})
    A = [1 << k for k in range(tot)]
    rng.shuffle(A)
    rest = A[1:r]
    rng.shuffle(rest)
    B = [A[r + 2]] + rest + [A[r + 3], A[r + 4], A[0], A[r + 0], A[r + 1]] + A[r + 5:]
    names = [("reg", r), ("lane", 5), ("warp", nw), ("block", nb)]

    def spec(v):
        bases, k = {}, 0
        for n, b in names:
            bases[n] = [tmp.unflatten(x) for x in v[k:k + b]]
            k += b
        return {"in_dims": names, "out_dims": out, "bases": bases}
    return {"A": spec(A), "B": spec(B), "elem_bytes": 2}


def test_convert_regs_trans_pairs():
    """Register-faithful conversions lowered with stmatrix.trans / ldmatrix
    (.trans), byte-exact; without the .trans tile these pairs have no
    register-faithful plan at all (the two sides' 4-byte words differ)."""
    rng = random.Random(1300)
    kinds = set()
    for _ in range(10):
        c = rand_trans_pair(rng, rng.randint(1, 6))
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        plan = ll.plan_describe(A, B, 16, "regs")
        if "regs" in plan:
            kinds.add((plan["regs"]["write"], plan["regs"]["read"]))
        batch = rng.choice([1, 2])
        src, dst = run_convert(c, path="regs", seed=rng.randint(0, 999), batch=batch)
        assert dst.tobytes() == expect_convert(c, src, batch).tobytes(), plan.get("regs")
    assert any("trans" in a or "trans" in b for a, b in kinds), kinds


def test_jit_failure_falls_back_to_template_kernels():
    """If NVRTC / module loading fails (forced by the jit_force_fail hook), the
    smem, shuffle and upcast paths run their template kernels from the
    library instead, byte-exact -- never a CPU path."""
    rng = random.Random(1400)
    ll.tune("jit_force_fail", 1)
    try:
        for w in (1, 2, 4):
            c = rand_pair(rng, 14, w)
            src, dst = run_convert(c, path="smem", seed=3, batch=2)
            assert dst.tobytes() == expect_convert(c, src, 2).tobytes()
        c = configs.cfg2(batch_bits=2)
        src, dst = run_convert(c, path="shuffle", seed=4)
        assert dst.tobytes() == expect_convert(c, src).tobytes()
        test_mxfp4_upcast(8, 7, "narrow")
    finally:
        ll.tune("jit_force_fail", 0)
