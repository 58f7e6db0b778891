"""Brute-force shared-memory bank-conflict counter -- oracle (tests only).

Model (P:679-689 and the Appendix lemma; reading A18/A23):
* shared memory has 32 banks of 4 bytes; byte address a lies in bank
  (a // 4) mod 32;
* a warp-level ld/st.shared instruction is issued for every (warp, value of
  the non-vector register bits); lane l accesses the 2^v elements given by the
  vector register bits, which must be contiguous and aligned in memory;
* "transactions involving more than 128 bytes will be split into multiple
  128-byte transactions": with granule g = 2^v . w bytes >= 4 the warp
  is split into phases of 128 / g consecutive lanes; sub-word granules form one
  phase of 32 lanes;
* a phase takes max over banks of the number of *distinct* 4-byte words it
  touches in that bank (same word = broadcast, no conflict); wavefronts of an
  instruction = sum over its phases.
"""

from . import f2


def smem_offsets(mem, dist):
    """offset(h) = S^{-1}(L(h)) for every flattened input index h of ``dist``.
    ``mem`` must be invertible (a memory layout)."""
    Sinv = f2.right_inverse(mem.cols, mem.out_bits)
    if len(mem.cols) != mem.out_bits:
        raise ValueError("memory layout must be square (invertible)")
    lcols = dist.cols
    return [f2.apply(Sinv, f2.apply(lcols, h)) for h in range(1 << dist.in_bits)]


def count_wavefronts(mem, dist, elem_bytes, vec_reg_bits, per_instruction=False):
    """Total wavefronts for accessing every element of ``dist`` once through
    the memory layout ``mem``.  ``vec_reg_bits`` lists, in element order, the
    register bits that form one vectorised access (may be empty)."""
    offs = smem_offsets(mem, dist)
    nreg = dist.in_size("reg")
    nlane = dist.in_size("lane") if dist.in_size("lane") else dist.in_size("thread")
    lane_name = "lane" if dist.in_size("lane") else "thread"
    nwarp = dist.in_size("warp")
    roff, loff, woff = dist.in_offset("reg"), dist.in_offset(lane_name), (
        dist.in_offset("warp") if nwarp or "warp" in dict(dist.in_dims) else None)
    v = len(vec_reg_bits)
    g = (1 << v) * elem_bytes
    other = [k for k in range(nreg) if k not in vec_reg_bits]
    lanes = 1 << nlane
    phase = max(1, 128 // g) if g >= 4 else lanes
    phase = min(phase, lanes)
    total = 0
    per = []
    for w in range(1 << nwarp):
        for o in range(1 << len(other)):
            rbase = 0
            for t, k in enumerate(other):
                if (o >> t) & 1:
                    rbase |= 1 << k
            words = []
            for l in range(lanes):
                h0 = (rbase << roff) | (l << loff) | ((w << woff) if nwarp else 0)
                base = offs[h0]
                if base % (1 << v):
                    raise ValueError("vector access is not aligned")
                for e in range(1 << v):
                    r = rbase
                    for t, k in enumerate(vec_reg_bits):
                        if (e >> t) & 1:
                            r |= 1 << k
                    h = (r << roff) | (l << loff) | ((w << woff) if nwarp else 0)
                    if offs[h] != base + e:
                        raise ValueError("vector elements are not contiguous in memory")
                words.append({(base * elem_bytes + b) // 4 for b in range(g)})
            wf = 0
            for p0 in range(0, lanes, phase):
                banks = {}
                for l in range(p0, p0 + phase):
                    for wd in words[l]:
                        banks.setdefault(wd % 32, set()).add(wd)
                wf += max(len(s) for s in banks.values())
            total += wf
            per.append(wf)
    return (total, per) if per_instruction else total


def lemma_wavefronts_per_instruction(mem_vect, mem_idx, lane_vecs, elem_bytes):
    """Appendix lemma: an access performs n.c wavefronts with
    n = 2^v . w / 4 >= 1 and c = |span(S_vect u S_idx) cap span(L_bank)|, where
    (reading A13) L_bank is the set of lane vectors of one 128-byte phase, i.e.
    L_thread without its last log2(n) vectors."""
    v = len(mem_vect)
    n = ((1 << v) * elem_bytes) // 4
    if n < 1:
        raise ValueError("lemma applies to granules of at least 4 bytes")
    drop = n.bit_length() - 1
    bank = list(lane_vecs[:len(lane_vecs) - drop]) if drop else list(lane_vecs)
    c = 1 << f2.intersection_dim(list(mem_vect) + list(mem_idx), bank)
    return n * c
