"""One-CTA in-kernel gather study (the analogue of fig:micro-gather).

For a row-major [M, K] fp32 tensor held in a blocked distributed layout (4
elements per thread along K, then lanes, warps, blocks), gather along K for
K = 32 ... 4096 with the warp-shuffle gather and the shared-memory gather,
timing the exchange in-kernel (ll_gather_timed: data already in registers /
shared memory, the exchange repeated `reps` times, clock64).  The shuffle
gather needs 2^|L_reg^axis| candidate shuffles per output (reading A19), so
its cost grows with K once the axis no longer fits one warp's lanes; the
shared-memory gather costs one ld.shared per output whatever K is.

Prints one JSON object: per K and path, cycles per repetition, elements of
the unit, warps used, warp-cycles per element, candidate shuffles, and
whether the paper's label criterion (L_warp^axis = L_block^axis = 0) holds.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2505_23819_b200 as ll
from oracle import convert as oconv
from oracle.layout import Layout as OL
from workloads.values import indices_torch, values_torch


def blocked_rowmajor(m_bits, k_bits):
    """reg k0,k1; lane k2..k6; warp k7..k9; block: the rest of k, then m."""
    out = [("m", m_bits), ("k", k_bits)]
    bits = [(0, 1 << j) for j in range(k_bits)] + [(1 << j, 0) for j in range(m_bits)]
    n = m_bits + k_bits
    dims = [("reg", 2), ("lane", 5), ("warp", 3), ("block", n - 10)]
    bases, p = {}, 0
    for nm, b in dims:
        bases[nm] = bits[p:p + b]
        p += b
    return {"in_dims": dims, "out_dims": out, "bases": bases}


def main():
    reps = int(os.environ.get("REPS", "64"))
    res = []
    for k_bits in range(5, 13):
        m_bits = 14 - k_bits if k_bits < 14 else 1
        spec = blocked_rowmajor(m_bits, k_bits)
        L = ll.Layout.from_spec(spec)
        n = 1 << L.in_bits
        src = values_torch(n, 3, 4, "cuda")
        idx = indices_torch(n, 4, 1 << k_bits, "cuda")
        exp = oconv.gather_np(src.cpu().numpy().view(np.uint32), idx.cpu().numpy(), OL(**spec), 1)
        for path in ("shuffle", "smem"):
            try:
                d = ll.gather_describe(L, 1, 32, path)
            except ll.LLError as e:
                res.append({"K": 1 << k_bits, "path": path, "unsupported": str(e)[:120]})
                continue
            # one CTA of 8 warps: 8 warp units (shuffle) or one CTA unit (smem)
            ub = d["warp_unit_bits"] if path == "shuffle" else d["cta_unit_bits"]
            elems = (8 << ub) if path == "shuffle" else (1 << ub)
            warps = 8
            out = torch.zeros_like(src)
            cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
            best = None
            for r in (reps, 2 * reps):
                vals = []
                for _ in range(5):
                    ll.gather_timed(src, idx, out, L, 1, 32, path, r, cyc)
                    torch.cuda.synchronize()
                    vals.append(int(cyc.item()))
                vals.sort()
                best = (best or []) + [(r, vals[len(vals) // 2])]
            ok = out.cpu().numpy().view(np.uint32)[:elems].tobytes() == exp[:elems].tobytes()
            # cycles per repetition from the slope between reps and 2 reps (drops fixed costs)
            (r1, c1), (r2, c2) = best
            per_rep = (c2 - c1) / (r2 - r1)
            res.append({"K": 1 << k_bits, "path": path, "elems_per_rep": elems, "warps": warps,
                        "cycles_per_rep": per_rep,
                        "warp_cycles_per_elem": per_rep * warps / elems,
                        "candidate_shuffles": d["candidate_shuffles"] if path == "shuffle" else None,
                        "paper_criterion": d["paper_criterion"], "parity_ok": ok})
    print(json.dumps({"reps": reps, "results": res}, indent=1))


if __name__ == "__main__":
    main()
