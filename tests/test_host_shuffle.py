"""Warp-shuffle conversion plans, host side (CPU only).

* the planner's paper sets I, E, F, G, R on the warp tile equal the oracle's
  step-by-step construction (oracle/shuffle.py) on the same load/store
  layouts;
* the per-round register / lane maps the kernel executes (alpha, beta,
  gamma, delta, eps, zeta and the elementary register operations) are
  simulated here, independently of the CUDA code, and deliver exactly the
  store layout's words; each round sends and receives one word per lane.
"""

import random

import pytest

import paper_2505_23819_b200 as ll
from oracle import shuffle as oshuffle
from oracle.layout import Layout as OLayout
from workloads import configs


def apply_ops(T, ops):
    for op, a, b in ops:
        T2 = []
        for k in range(len(T)):
            if op == 0:
                ba, bb = (k >> a) & 1, (k >> b) & 1
                kk = k ^ ((1 << a) | (1 << b)) if ba != bb else k
            else:
                kk = k ^ (1 << b) if (k >> a) & 1 else k
            T2.append(T[kk])
        T = T2
    return T


def lane_mask(cols, l):
    m = 0
    for c in range(5):
        if (l >> c) & 1:
            m ^= cols[c]
    return m


def simulate(sh):
    Aw, Al, Bw, Bl = sh["word_bits_ld"], sh["lanes_ld"], sh["word_bits_st"], sh["lanes_st"]
    LB = len(Aw)
    NW = 1 << LB

    def vec(wbits, lbits, q, l):
        x = 0
        for b in range(LB):
            if (q >> b) & 1:
                x ^= wbits[b]
        for c in range(5):
            if (l >> c) & 1:
                x ^= lbits[c]
        return x

    regs = [[vec(Aw, Al, q, l) for q in range(NW)] for l in range(32)]
    S = []
    for l in range(32):
        beta = lane_mask(sh["beta_lane"], l)
        R1 = [regs[l][m ^ beta] for m in range(NW)]
        S.append(apply_ops(R1, sh["pre_ops"]))
    Q = []
    for l in range(32):
        delta = lane_mask(sh["delta_lane"], l)
        X = [S[sh["gamma"][k] ^ delta][k] for k in range(NW)]
        Y = apply_ops(X, sh["post_ops"])
        zeta = lane_mask(sh["zeta_lane"], l)
        Q.append([Y[m ^ zeta] for m in range(NW)])
    want = [[vec(Bw, Bl, q, l) for q in range(NW)] for l in range(32)]
    return Q == want


def rand_spec(rng, d, w):
    vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
    names = [("reg", vb + rng.randint(0, 2)), ("lane", 5)]
    rest = d - names[0][1] - 5
    nw = min(rest, rng.randint(0, 2))
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
    return specs


def oracle_sets(d, sh):
    """The oracle's construction on the plan's word-level warp tile."""
    n = max(x.bit_length() for x in sh["word_bits_ld"] + sh["lanes_ld"])
    A = OLayout([("reg", len(sh["word_bits_ld"])), ("lane", 5)], [("t", n)],
                {"reg": [(x,) for x in sh["word_bits_ld"]], "lane": [(x,) for x in sh["lanes_ld"]]})
    B = OLayout([("reg", len(sh["word_bits_st"])), ("lane", 5)], [("t", n)],
                {"reg": [(x,) for x in sh["word_bits_st"]], "lane": [(x,) for x in sh["lanes_st"]]})
    # payload 32 bits, one word per shuffle: elements here are whole words (w = 4)
    return oshuffle.shuffle_plan(A, B, 4), A, B


@pytest.mark.parametrize("name,c", [("cfg1a", configs.cfg1("mma")), ("cfg1b", configs.cfg1("T")),
                                    ("cfg2", configs.cfg2(batch_bits=2)),
                                    ("cfg5", configs.cfg5(m_bits=8, kb_bits=7))])
def test_shuffle_plan_configs(name, c):
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    d = ll.plan_describe(A, B, 8 * c["elem_bytes"], "shuffle")
    assert d["path"] == "shuffle"
    sh = d["shuffle"]
    assert sh["ok"]
    op, Ao, Bo = oracle_sets(d, sh)
    assert op["I"] == sh["I"] and op["E"] == sh["E"] and op["F"] == sh["F"]
    assert op["G"] == sh["G"] and op["R"] == sh["R"]
    assert op["rounds"] == sh["rounds"]
    assert oshuffle.simulate(Ao, Bo, op)["ok"]          # the paper's rounds realise B
    assert simulate(sh)                                  # the kernel's maps realise B


@pytest.mark.parametrize("w", [1, 2, 4])
def test_shuffle_plan_random_pairs(w):
    rng = random.Random(400 + w)
    done = 0
    while done < 25:
        d = rng.randint(11, 15)
        sa, sb = rand_spec(rng, d, w)
        A, B = ll.Layout.from_spec(sa), ll.Layout.from_spec(sb)
        try:
            desc = ll.plan_describe(A, B, 8 * w, "shuffle")
        except ll.LLError:
            continue
        sh = desc["shuffle"]
        op, Ao, Bo = oracle_sets(desc, sh)
        assert op["R"] == sh["R"] and op["G"] == sh["G"]
        assert simulate(sh)
        done += 1


def test_shuffle_infeasible_for_transpose():
    """A transpose's exchange spans several warps: (B^-1 o A)_warp != id."""
    c = configs.cfg3(n_bits=7)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    with pytest.raises(ll.LLError) as e:
        ll.plan_describe(A, B, 16, "shuffle")
    assert e.value.name == "LL_ERR_UNSUPPORTED"
