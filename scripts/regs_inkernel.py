"""In-kernel cost of one register -> smem -> register conversion on the
register-faithful path (the paper's microbenchmark view: one CTA, the
conversion inside the kernel).  For each case the exchange is
repeated `reps` times inside the kernel; cycles/conversion = (cycles(reps) -
cycles(1)) / (reps - 1), median over trials.  Compares stmatrix/ldmatrix
(regs_matrix=1) against vectorised st/ld.shared only (regs_matrix=0).

    python scripts/regs_inkernel.py > profiles/.../regs_inkernel.json
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402


def measure(c, mat, reps=1024, trials=7):
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    ll.tune("regs_matrix", mat)
    plan = ll.plan_describe(A, B, 8 * w, "regs")
    n = 1 << A.in_bits
    src = values_torch(n, 3, w, "cuda")
    dst = torch.empty_like(src)
    cy = torch.zeros(1024, dtype=torch.int64, device="cuda")
    per = []
    for _ in range(trials):
        res = []
        for r in (1, reps):
            ll.convert_regs_timed(src, A, dst, B, 8 * w, reps=r, cycles=cy)
            torch.cuda.synchronize()
            res.append(int(cy[0].item()))
        per.append((res[1] - res[0]) / (reps - 1))
    ll.tune("regs_matrix", 1)
    return {"cycles_per_conversion": statistics.median(per), "plan": plan["regs"],
            "granule_bytes": plan["granule_bytes"],
            "pred_wavefronts": [plan["pred_wavefronts_per_sts"], plan["pred_wavefronts_per_lds"]]}


def main():
    cases = [("cfg1a Fig.1 A -> mma C (2 warps, fp16)", configs.cfg1("mma")),
             ("cfg1b Fig.1 A -> A^T (2 warps, fp16)", configs.cfg1("T")),
             ("cfg2 one 128x128 tile: mma C -> blocked (4 warps, fp16)", configs.cfg2(batch_bits=0))]
    out = []
    for name, c in cases:
        row = {"case": name}
        for mat in (1, 0):
            row["matrix" if mat else "vector_only"] = measure(c, mat)
        out.append(row)
    print(json.dumps({"what": __doc__.strip().splitlines()[0], "sm_clock_note": "cycles = SM clock64",
                      "rows": out}, indent=1))


if __name__ == "__main__":
    main()
