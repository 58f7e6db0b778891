"""One small launch of every device path, each checked against the oracle --
the workload for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python scripts/sanitize_paths.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from oracle import convert as oconv  # noqa: E402
from oracle.layout import Layout as OL  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import indices_torch, values_torch  # noqa: E402

NP = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


def conv(c, path, batch=1):
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = (1 << A.in_bits) * batch
    src = values_torch(n, 3, w, "cuda")
    dst = torch.zeros((1 << B.in_bits) * batch, dtype=src.dtype, device="cuda")
    ll.convert(src, A, dst, B, 8 * w, path=path, batch=batch)
    torch.cuda.synchronize()
    s = src.cpu().numpy().view(NP[w])
    nA = A.in_bits
    exp = np.concatenate([oconv.convert_np(s[b << nA:(b + 1) << nA], OL(**c["A"]), OL(**c["B"]))
                          for b in range(batch)])
    ok = dst.cpu().numpy().view(NP[w]).tobytes() == exp.tobytes()
    print("%-10s %-16s %s" % (c["name"], path, "ok" if ok else "MISMATCH"), flush=True)
    return ok


def main():
    ok = True
    ok &= conv(configs.cfg2(batch_bits=2), "smem")
    ok &= conv(configs.cfg3(n_bits=8), "smem")
    ok &= conv(configs.cfg5(m_bits=8, kb_bits=8), "smem")
    ok &= conv(configs.cfg2(batch_bits=2), "shuffle")
    ok &= conv(configs.cfg2(batch_bits=2), "smem_async")
    ok &= conv(configs.cfg3(n_bits=8), "smem_tma")
    ok &= conv(configs.cfg5(m_bits=8, kb_bits=8), "smem_tma")
    ok &= conv(configs.cfg3(n_bits=8), "smem_tma_store")
    ok &= conv(configs.cfg1("mma"), "regs")
    ok &= conv(configs.cfg2(batch_bits=1), "regs")
    ok &= conv(configs.cfg2w(batch_bits=1), "regs_shuffle")
    ok &= conv(configs.cfg2(batch_bits=1), "generic")
    # ldmatrix / stmatrix .trans (register-faithful transposed fragments)
    import random
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import rand_trans_pair  # noqa: E402
    ok &= conv(dict(rand_trans_pair(random.Random(3), 3), name="trans"), "regs")
    # round 2: compiled TMA kernels (non-persistent default and persistent
    # rings), register permutation, small-granule shuffle (config 6), the
    # b8 matrix tiles, broadcast dedup
    ok &= conv(configs.cfg2(batch_bits=2), "smem_tma")
    ok &= conv(configs.cfg2(batch_bits=2), "smem_tma_store")
    ll.tune("tmaj_tpc", -1)
    ok &= conv(configs.cfg5(m_bits=9, kb_bits=8), "smem_tma")
    ok &= conv(configs.cfg5(m_bits=9, kb_bits=8), "smem_tma_store")
    ll.tune("tmaj_tpc", 0)
    ok &= conv(configs.cfg6(n_bits=7, k_bits=7), "auto")
    from test_gpu_parity import perm_pair, b8_pair, _bcast_pair  # noqa: E402
    ok &= conv(dict(perm_pair(random.Random(5), 14, 2, 4, "reg"), name="regperm"), "regperm")
    for kind in ("both", "st_vec", "ld_vec"):
        ok &= conv(dict(b8_pair(random.Random(6), kind, nr=4, nw=1), name="b8_" + kind), "regs")
    ok &= conv(dict(_bcast_pair(random.Random(7), 13, 2, 0, 2), name="bcast"), "smem")
    # session 3: PDL prologue prefetch in every CTA, the diagonal tile order,
    # the register permutation's prefetch, the direct gather (AUTO is the
    # smem gather now), the upcast with PDL (defaults cover the first-wave
    # prefetch and the shuffle / gather PDL)
    ll.tune("pdl_prefetch", 2)
    ok &= conv(configs.cfg3(n_bits=8), "smem")
    ll.tune("pdl_prefetch", 1)
    ll.tune("tile_xor", 3)
    ok &= conv(configs.cfg3(n_bits=8), "smem")
    ll.tune("tile_xor", 0)
    ll.tune("regperm_prefetch", 1)
    ok &= conv(dict(perm_pair(random.Random(5), 14, 2, 4, "reg"), name="regperm_pf"), "regperm")
    ll.tune("regperm_prefetch", 0)
    # the template smem kernel (the default compiles the plan)
    ll.tune("smem_jit", 0)
    ok &= conv(configs.cfg3(n_bits=8), "smem")
    ll.tune("smem_jit", 1)
    g = configs.cfg4(r_bits=3)
    L = ll.Layout.from_spec(g["L"])
    m = 1 << L.in_bits
    for path in ("shuffle", "smem", "auto", "generic"):
        gs = values_torch(m, 4, 4, "cuda")
        gi = indices_torch(m, 5, 32, "cuda")
        go = torch.empty_like(gs)
        ll.gather(gs, gi, go, L, g["axis"], 32, path=path)
        torch.cuda.synchronize()
        exp = oconv.gather_np(gs.cpu().numpy().view(np.uint32), gi.cpu().numpy(), OL(**g["L"]), 2)
        good = go.cpu().numpy().view(np.uint32).tobytes() == exp.tobytes()
        print("%-10s %-16s %s" % ("cfg4", "gather " + path, "ok" if good else "MISMATCH"), flush=True)
        ok &= good
    # fused mxfp4 upcast (NEXT 1) against oracle.mxfp4.upcast_np
    from oracle import mxfp4 as omx
    c = configs.cfg5(m_bits=8, kb_bits=7)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    packed = values_torch(n, 9, 1, "cuda")
    sc = (indices_torch((1 << 8) * (1 << 3), 10, 16, "cuda") + 120).to(torch.uint8)
    exp = omx.upcast_np(packed.cpu().numpy(), OL(**c["A"]), sc.cpu().numpy(), OL(**c["B"]))
    for pdl in (0, 1):
        ll.tune("upcast_pdl", pdl)
        out = torch.empty(2 * n, dtype=torch.int16, device="cuda")
        ll.mxfp4_upcast(packed, A, sc, out, B)
        torch.cuda.synchronize()
        good = out.cpu().numpy().view(np.uint16).tobytes() == exp.tobytes()
        print("%-10s %-16s %s" % ("cfg5", "mxfp4_upcast" + " pdl" * pdl, "ok" if good else "MISMATCH"), flush=True)
        ok &= good
    ll.tune("upcast_pdl", 0)
    print("ALL OK" if ok else "FAILURES")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
