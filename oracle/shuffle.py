"""Intra-warp data exchange by warp shuffles -- oracle (tests only).

``shuffle_plan`` follows "Intra-warp Data Exchange" step by step:
V (vectorisation, <= 32-bit payload), I = A_thread cap B_thread,
E = A_thread \\ I, F = B_thread \\ I (ascending), G = {e_i xor f_i},
R completes V u I u G to a basis of the warp-local space; round i exchanges
the affine space R(i) xor span(V u I u G).  ``simulate`` executes the
rounds on a software register file and checks the paper's claims (one vector
sent and one received per thread per round, 2^|R| rounds, final placement =
B).  Preconditions of the paper: (B^{-1} o A)_warp is the identity
and no broadcasting.
"""

import math

from . import f2


def _lane(L):
    return L.sub("lane") if L.in_size("lane") else L.sub("thread")


def _lane_name(L):
    return "lane" if L.in_size("lane") else "thread"


def shuffle_plan(A, B, elem_bytes, payload_bits=32):
    for L in (A, B):
        if any(x == 0 for x in L.cols):
            raise ValueError("shuffle_plan: broadcasting is excluded (P:625)")
    if sorted(A.sub("warp")) != sorted(B.sub("warp")):
        raise ValueError("shuffle_plan: warp part differs; shuffles need (B^-1 o A)_warp = id (P:624)")
    # 1. vectorisation size: V within A_reg cap B_reg, one shuffle payload
    breg = set(B.sub("reg"))
    common = [x for x in A.sub("reg") if x in breg]
    vmax = int(math.log2(max(1, (payload_bits // 8) // elem_bytes))) if elem_bytes * 8 <= payload_bits else 0
    V = common[:vmax]
    # 2. tiling and exchange
    At, Bt = _lane(A), _lane(B)
    I = sorted(x for x in At if x in Bt)
    E = sorted(x for x in At if x not in I)
    F = sorted(x for x in Bt if x not in I)
    if len(E) != len(F):
        raise ValueError("shuffle_plan: |E| != |F| (broadcasting?)")
    G = [e ^ f for e, f in zip(E, F)]
    # R: extend V u I u G to a basis of the warp-local space span(A_reg u A_thread),
    # lowest standard vectors first (reading A9)
    local = A.sub("reg") + At
    span_local = sorted(local)                 # unit vectors: a coordinate subspace
    base = V + I + G
    R = []
    for e in sorted(span_local):
        if not f2.in_span(e, base + R):
            R.append(e)
    if f2.rank(base + R) != len(local):
        raise ValueError("shuffle_plan: basis completion failed")
    return dict(V=V, I=I, E=E, F=F, G=G, R=R, rounds=1 << len(R))


def round_set(plan, i):
    """R(i) xor span(V u I u G)."""
    Ri = 0
    for k, r in enumerate(plan["R"]):
        if (i >> k) & 1:
            Ri ^= r
    return {Ri ^ x for x in f2.span(plan["V"] + plan["I"] + plan["G"])}


def simulate(A, B, plan, warp=0):
    """Execute the rounds of ``plan`` for one warp on a register file.

    Returns dict(ok, rounds, sends_per_round) after checking, for every round,
    that each lane sends exactly one vector and receives exactly one vector
     and that the final registers hold B's placement."""
    ln = _lane_name(A)
    nreg, nlane = A.in_size("reg"), A.in_size(ln)
    regA = {}   # tensor element -> (lane, reg) under A, for this warp
    for l in range(1 << nlane):
        for r in range(1 << nreg):
            x = f2.apply(A.cols, (r << A.in_offset("reg")) | (l << A.in_offset(ln))
                         | (warp << A.in_offset("warp") if A.in_size("warp") else 0))
            regA[x] = (l, r)
    posB = {}
    for l in range(1 << nlane):
        for r in range(1 << nreg):
            x = f2.apply(B.cols, (r << B.in_offset("reg")) | (l << B.in_offset(ln))
                         | (warp << B.in_offset("warp") if B.in_size("warp") else 0))
            posB[x] = (l, r)
    Vspan = f2.span(plan["V"])
    stateA = {pos: x for x, pos in regA.items()}   # register file before the exchange
    stateB = {}
    covered = []
    per_round = []
    for i in range(plan["rounds"]):
        S = round_set(plan, i)
        sends = {}
        recvs = {}
        for x in S:
            # the vector (coset of span V) containing x, sent by its A-lane
            la, _ = regA[x]
            lb, _ = posB[x]
            rep = min(x ^ y for y in Vspan)
            sends.setdefault(la, set()).add(rep)
            recvs.setdefault(lb, set()).add(rep)
            stateB[posB[x]] = stateA[regA[x]]   # lane la sends, lane lb receives
            covered.append(x)
        ok_round = (len(sends) == 1 << nlane and len(recvs) == 1 << nlane
                    and all(len(s) == 1 for s in sends.values())
                    and all(len(s) == 1 for s in recvs.values()))
        per_round.append(ok_round)
    final_ok = (all(stateB.get(posB[x]) == x for x in posB)
                and sorted(covered) == sorted(posB))   # rounds partition the warp space
    return dict(ok=final_ok and all(per_round), rounds=plan["rounds"],
                rounds_ok=per_round, final_ok=final_ok)
