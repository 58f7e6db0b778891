"""Shared-memory instruction counts of conversions between broadcast layouts
(the analogue of tab:micro-broadcasting): dedup vs naive.

The paper counts shared-memory instructions of Triton kernels on layouts
with duplicated data (replicated warps / threads / registers when the layout
tile exceeds the tensor, and sliced layouts) on the
shapes [128,16], [128,128], [32,128], [32,32], [16,16] with 4 warps.  Here
each shape is a batch of 256 CTA tiles ([256, M, N], block bits = the batch
dim), converted between two layouts of one family on B200:

  Blocked          blocked(spt [1,8], tpw [4,8], wpc [4,1]) -> blocked(spt [4,1], tpw [8,4], wpc [1,4])
  MMA              mma m16n8 accumulator (4 warps along M)  -> blocked(spt [1,8], ...)
  Sliced<Blocked>  slice(blocked, N)                        -> slice(blocked', N)
  Sliced<MMA>      slice(mma, N)                            -> slice(blocked, N)

dedup = the default plan (each distinct element crosses shared memory once,
copies made in registers / by extra stores); naive = knob bcast_dedup=0
(destination copies re-run the exchange as separate tiles; copies inside
16-byte vectors fall to the element-wise kernel, which uses no shared memory).
Counts are ncu's smsp__sass_inst_executed_op_shared_{st,ld}.sum per launch,
taken in this script's own ncu subprocess; every conversion is checked
against the oracle first.

    python scripts/bcast_smem_counts.py > out.json      (needs ncu and a GPU)
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(7, 4), (7, 7), (5, 7), (5, 5), (4, 4)]      # log2 of [128,16] [128,128] [32,128] [32,32] [16,16]
BATCH_BITS = 8


def _bit(out, name, k):
    return tuple((1 << k) if d == name else 0 for d, _ in out)


def triton_blocked(mb, nb, spt, tpw, wpc, order):
    """Triton's blocked layout on [2^BATCH_BITS, 2^mb, 2^nb] (one CTA tile per
    batch index): reg, lane, warp bits per dim in `order` (fastest first);
    tile bits beyond a dim are zero columns (replication), dims larger than
    the tile get extra register bits."""
    out = [("b", BATCH_BITS), ("i", mb), ("j", nb)]
    size = {"i": mb, "j": nb}
    used = {"i": 0, "j": 0}
    names = ["i", "j"]
    bases = {"reg": [], "lane": [], "warp": []}
    lg = lambda v: [x.bit_length() - 1 for x in v]  # noqa: E731  (sizes are powers of two)
    for lab, per in (("reg", lg(spt)), ("lane", lg(tpw)), ("warp", lg(wpc))):
        for o in order:
            d = names[o]
            for _ in range(per[o]):
                if used[d] < size[d]:
                    bases[lab].append(_bit(out, d, used[d]))
                    used[d] += 1
                else:
                    bases[lab].append(tuple(0 for _ in out))
    for o in order:
        d = names[o]
        while used[d] < size[d]:
            bases["reg"].append(_bit(out, d, used[d]))
            used[d] += 1
    bases["block"] = [_bit(out, "b", k) for k in range(BATCH_BITS)]
    dims = [(n, len(bases[n])) for n in ("reg", "lane", "warp", "block")]
    return {"in_dims": dims, "out_dims": out, "bases": bases}


def mma_out(mb, nb):
    """mma.sync m16n8 accumulator tile, 4 warps along M, repeated in registers;
    rows / columns beyond the tensor are zero columns."""
    out = [("b", BATCH_BITS), ("i", mb), ("j", nb)]
    z = tuple(0 for _ in out)

    def b(d, k):
        return _bit(out, d, k) if k < {"i": mb, "j": nb}[d] else z
    bases = {"reg": [b("j", 0), b("i", 3)], "lane": [b("j", 1), b("j", 2), b("i", 0), b("i", 1), b("i", 2)],
             "warp": [b("i", 4), b("i", 5)]}
    for k in range(3, nb):
        bases["reg"].append(b("j", k))
    for k in range(6, mb):
        bases["reg"].append(b("i", k))
    bases["block"] = [_bit(out, "b", k) for k in range(BATCH_BITS)]
    dims = [(n, len(bases[n])) for n in ("reg", "lane", "warp", "block")]
    return {"in_dims": dims, "out_dims": out, "bases": bases}


def sliced(spec, dim):
    axis = [d for d, _ in spec["out_dims"]].index(dim)
    out = [d for i, d in enumerate(spec["out_dims"]) if i != axis]
    bases = {n: [tuple(c for i, c in enumerate(v) if i != axis) for v in vs] for n, vs in spec["bases"].items()}
    return {"in_dims": spec["in_dims"], "out_dims": out, "bases": bases}


def cases():
    out = []
    for mb, nb in SHAPES:
        A_bl = triton_blocked(mb, nb, [1, 8], [4, 8], [4, 1], [1, 0])
        B_bl = triton_blocked(mb, nb, [4, 1], [8, 4], [1, 4], [0, 1])
        mm = mma_out(mb, nb)
        shape = "[%d,%d]" % (1 << mb, 1 << nb)
        out.append(("Blocked", shape, A_bl, B_bl))
        out.append(("MMA", shape, mm, A_bl))
        out.append(("Sliced<Blocked>", shape, sliced(A_bl, "j"), sliced(B_bl, "j")))
        out.append(("Sliced<MMA>", shape, sliced(mm, "j"), sliced(A_bl, "j")))
    return out


def child():
    import numpy as np
    import torch
    import paper_2505_23819_b200 as ll
    from oracle import convert as oconv
    from oracle.layout import Layout as OL
    from workloads.values import values_torch
    info = []
    for fam, shape, a, b in cases():
        A, B = ll.Layout.from_spec(a), ll.Layout.from_spec(b)
        src = values_torch(1 << A.in_bits, 9, 2, "cuda")
        dst = torch.zeros(1 << B.in_bits, dtype=torch.int16, device="cuda")
        rec = {"family": fam, "shape": shape, "src_elems": 1 << A.in_bits, "dst_elems": 1 << B.in_bits}
        exp = oconv.convert_np(src.cpu().numpy().view(np.uint16), OL(**a), OL(**b))
        for mode in (1, 0):
            ll.tune("bcast_dedup", mode)
            d = ll.plan_describe(A, B, 16)
            ll.convert(src, A, dst, B, 16)
            torch.cuda.synchronize()
            ok = dst.cpu().numpy().view(np.uint16).tobytes() == exp.tobytes()
            rec["dedup" if mode else "naive"] = {"path": d["path"], "parity_ok": ok,
                                                 "bcast_dedup": d.get("bcast_dedup")}
        ll.tune("bcast_dedup", 1)
        info.append(rec)
    with open(os.environ["BCAST_INFO"], "w") as f:
        json.dump(info, f)


def main():
    info_path = "/tmp/bcast_info.json"
    metrics = ["smsp__sass_inst_executed_op_shared_st.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
               "gpu__time_duration.sum"]
    env = dict(os.environ, BCAST_INFO=info_path)
    cmd = ["ncu", "--metrics", ",".join(metrics), "--clock-control", "none", "--csv", "--page", "raw",
           "--kernel-name", "regex:(ll_smem|convert_.*kernel)", sys.executable, os.path.abspath(__file__),
           "--child"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, vals = rows[0], rows[2:]
    info = json.load(open(info_path))
    res, k = [], 0
    for rec in info:
        for mode in ("dedup", "naive"):
            r = vals[k]
            k += 1
            rec[mode].update({
                "kernel": r[hdr.index("Kernel Name")][:40],
                "sts": float(r[hdr.index(metrics[0])].replace(",", "")),
                "lds": float(r[hdr.index(metrics[1])].replace(",", "")),
                "us": float(r[hdr.index(metrics[2])].replace(",", "")) / 1000.0})
        d, n = rec["dedup"], rec["naive"]
        rec["sts_reduction"] = (1 - d["sts"] / n["sts"]) if n["sts"] else None
        res.append(rec)
    print(json.dumps({"rows": res, "ncu_rc": p.returncode}, indent=1))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        main()
