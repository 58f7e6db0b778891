"""Diagnose the compiled TMA kernels at full size: mismatches against the
AUTO path's output (itself oracle-verified by the GPU suite) under knobs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402

VARIANTS = [{}, {"tmaj_fence": 0}, {"tmaj_fence": 0, "tmaj_late": 1}, {"tmaj_stages": 2}, {"pdl": 0},
            {"tmaj_cps": 2}, {"tmaj_k": 1}, {"tma_jit": 0}]


def main():
    out = []
    for name, c in (("cfg2", configs.cfg2()), ("cfg5", configs.cfg5()), ("cfg3", configs.cfg3())):
        w = c["elem_bytes"]
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        src = values_torch(1 << A.in_bits, 17, w, "cuda")
        ref = torch.empty(1 << B.in_bits, dtype=src.dtype, device="cuda")
        ll.convert(src, A, ref, B, 8 * w)
        d = ll.plan_describe(A, B, 8 * w, "smem_tma")
        tile_elems = 1 << len(d["tile_dst_bits"])
        for path in ("smem_tma", "smem_tma_store"):
            for v in VARIANTS:
                for k, x in v.items():
                    ll.tune(k, x)
                res = []
                for rep in range(3):
                    dst = torch.zeros_like(ref)
                    ll.convert(src, A, dst, B, 8 * w, path=path)
                    torch.cuda.synchronize()
                    bad = (dst != ref).nonzero().flatten()
                    res.append({"mismatch": int(bad.numel()),
                                "first": bad[:4].tolist(),
                                "zeros_in_bad": int((dst[bad] == 0).sum().item()) if bad.numel() else 0})
                for k in v:
                    ll.tune(k, {"pdl": 1, "tmaj_fence": 1, "tma_jit": 1}.get(k, 0))
                out.append({"cfg": name, "path": path, "knobs": v, "runs": res, "tile_elems": tile_elems})
                print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
