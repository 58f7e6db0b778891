"""Optimal swizzling -- oracle (tests only).

``optimal_swizzle`` follows the paper's construction step by step, in its
order and notation: main text "Optimal Swizzling" and Appendix
"Choosing a Basis for Bank Indices".  Readings:
A13 (P built from A_bank/B_bank, the main-text rule), A14 (Appendix names
S_vect/S_bank/S_idx, l), A15 (select H first, then C), A16 (pad from A_bank in
ascending order).  ``brute_force_min_wavefronts`` searches all index
subspaces for tiny d, to check optimality against the bank counter.

Vectors are flat tensor indices (ints, LSB-first); A and B are distributed
layouts over the same tensor with input dims reg / lane / warp.
"""

import itertools
import math

from . import f2
from .layout import Layout, from_flat


def _lane(L):
    return L.sub("lane") if L.in_size("lane") else L.sub("thread")


def vector_set(A, B, elem_bytes, max_vec_bytes=16):
    """V: a basis of A_reg cap B_reg ("choosing a basis of A_reg cap B_reg
    as done for warp shuffles"), capped at ``max_vec_bytes`` of one vectorised
    ld/st.shared, taken in A's register order."""
    breg = set(x for x in B.sub("reg") if x)
    cand = [x for x in A.sub("reg") if x and x in breg]
    vmax = int(math.log2(max(1, max_vec_bytes // elem_bytes)))
    return cand[:vmax]


def optimal_swizzle(A, B, elem_bytes, V=None, variant="main", max_vec_bytes=16):
    """Return (S, info): S is the memory layout offset -> tensor whose columns
    are [S_vect | S_bank | S_idx] (P:673-677 / P:1075-1079), and ``info``
    records the intermediate sets of the construction."""
    d = A.out_bits
    if V is None:
        V = vector_set(A, B, elem_bytes, max_vec_bytes)
    v = len(V)
    # b = log2(128 / (2^v w))
    b = int(math.log2(128 // ((1 << v) * elem_bytes))) if (1 << v) * elem_bytes <= 128 else 0
    b = min(b, d - v)
    ell = d - v - b
    At, Bt = [x for x in _lane(A) if x], [x for x in _lane(B) if x]
    if variant == "main":
        # "taking out the last few log2 max(1, 2^v w / 4) vectors"
        drop = int(math.log2(max(1, ((1 << v) * elem_bytes) // 4)))
        Abank = At[:len(At) - drop] if drop else At
        Bbank = Bt[:len(Bt) - drop] if drop else Bt
    else:  # Appendix: A_thread / B_thread
        Abank, Bbank = At, Bt
    # P = span(S_vect u A_bank) u span(S_vect u B_bank)
    # E = A_bank \ B_bank, F = B_bank \ A_bank; |E| <= |F| w.l.o.g.
    E = sorted(x for x in Abank if x not in Bbank)
    F = sorted(x for x in Bbank if x not in Abank)
    if len(E) > len(F):
        E, F = F, E
    H = [e ^ f for e, f in zip(E, F)]
    # C: complement of span(P)
    C = f2.complete_basis(_basis_of(list(V) + Abank + Bbank), d)
    # choose S_idx
    if len(H) + len(C) >= ell:
        idx = (H + C)[:ell]
        unavoidable = False
    else:
        idx = H + C
        for x in Abank:                                   # reading A16
            if len(idx) == ell:
                break
            if not f2.in_span(x, list(V) + idx):
                idx.append(x)
        unavoidable = True
    # S_bank completes S_vect u S_idx to a basis of F2^d
    bank = f2.complete_basis(list(V) + idx, d)
    cols = list(V) + bank + idx
    S = from_flat([("offset", d)], A.out_dims, cols)
    info = dict(V=list(V), v=v, b=b, ell=ell, A_bank=Abank, B_bank=Bbank, E=E, F=F,
                H=H, C=C, S_idx=idx, S_bank=bank, unavoidable=unavoidable)
    return S, info


def _basis_of(vectors):
    out = []
    for x in vectors:
        if x and not f2.in_span(x, out):
            out.append(x)
    return out


def abstract_lemma_dim(U, V, d):
    """Appendix abstract swizzling lemma: the largest subspace
    with trivial intersection with U u V has dimension d - max(dim U, dim V)."""
    return d - max(f2.rank(U), f2.rank(V))


def brute_force_max_trivial_dim(U, V, d):
    """Largest dim of a subspace W of F2^d with W cap (span U u span V) = {0}
    (brute force over all subspaces; d <= 5)."""
    su, sv = f2.span(U), f2.span(V)
    bad = (su | sv) - {0}
    best = 0
    nonzero = [x for x in range(1, 1 << d) if x not in bad]
    for k in range(1, d + 1):
        found = False
        for combo in itertools.combinations(nonzero, k):
            if f2.rank(list(combo)) != k:
                continue
            if not (f2.span(list(combo)) - {0}) & bad:
                found = True
                break
        if not found:
            break
        best = k
    return best


def vec_reg_bits(L, V):
    """Register bits of L holding the vectors of V, in V's order."""
    regs = L.sub("reg")
    return [regs.index(x) for x in V]


def swizzle_wavefronts(S, A, B, elem_bytes, V):
    """(write wavefronts storing A, read wavefronts loading B) through S."""
    from . import banks
    wa = banks.count_wavefronts(S, A, elem_bytes, vec_reg_bits(A, V))
    wb = banks.count_wavefronts(S, B, elem_bytes, vec_reg_bits(B, V))
    return wa, wb


def brute_force_min_wavefronts(A, B, elem_bytes, V):
    """Minimum over all choices of S_idx (S_vect = V fixed, S_bank completed)
    of write + read wavefronts, by exhaustive search (tiny d only)."""
    d = A.out_bits
    v = len(V)
    b = int(math.log2(128 // ((1 << v) * elem_bytes)))
    b = min(b, d - v)
    ell = d - v - b
    # vectorised accesses need S_idx free of S_vect components (aligned vectors)
    vmask = 0
    for x in V:
        vmask |= x
    cands = [x for x in range(1, 1 << d) if not x & vmask]
    seen = set()
    best = None
    for combo in itertools.combinations(cands, ell):
        allv = list(V) + list(combo)
        if f2.rank(allv) != len(allv):
            continue
        key = frozenset(f2.span(list(combo)))
        if key in seen:
            continue
        seen.add(key)
        bank = f2.complete_basis(allv, d)
        S = from_flat([("offset", d)], A.out_dims, list(V) + bank + list(combo))
        wa, wb = swizzle_wavefronts(S, A, B, elem_bytes, V)
        if best is None or wa + wb < best:
            best = wa + wb
    return best
