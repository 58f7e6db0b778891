"""In-kernel cost of fp8 register-faithful conversions lowered with the
sm_100a 8-bit matrix tiles (stmatrix.m16n8.trans.b8 / ldmatrix.m16n16.
trans.b8) vs the plan the planner makes without them (knob
regs_b8=0: vector st/ld.shared or b16 matrices, where one exists).  One CTA,
the register -> smem -> register exchange repeated inside the kernel;
cycles/conversion = (cycles(reps) - cycles(1)) / (reps - 1), median of trials.

    python scripts/b8_inkernel.py > out.json
"""
import json
import os
import random
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from tests.test_gpu_parity import b8_pair  # noqa: E402
from workloads.values import values_torch  # noqa: E402


def measure(c, reps=512, trials=7):
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    ll.tune("regs_shuffle_max_rounds", 0)
    try:
        plan = ll.plan_describe(A, B, 8, "regs")
    except ll.LLError as e:
        return {"unsupported": str(e)[:100]}
    n = 1 << A.in_bits
    src = values_torch(n, 3, 1, "cuda")
    dst = torch.empty_like(src)
    cy = torch.zeros(1024, dtype=torch.int64, device="cuda")
    per = []
    for _ in range(trials):
        res = []
        for r in (1, reps):
            ll.convert_regs_timed(src, A, dst, B, 8, reps=r, cycles=cy)
            torch.cuda.synchronize()
            res.append(int(cy[0].item()))
        per.append((res[1] - res[0]) / (reps - 1))
    r = plan["regs"]
    return {"cycles_per_conversion": statistics.median(per), "write": r["write"], "write_words": r["write_words"],
            "read": r["read"], "read_words": r["read_words"],
            "instr_per_thread": [r["write_instr_per_thread"], r["read_instr_per_thread"]]}


def main():
    rng = random.Random(2025)
    rows = []
    for kind in ("both", "st_vec", "ld_vec"):
        for nr, nw in ((3, 1), (4, 1), (4, 2), (5, 1), (5, 2)):
            for _ in range(2):
                c = b8_pair(rng, kind, nr=nr, nw=nw, nb=0)
                row = {"kind": kind, "reg_bits": nr, "warps_log2": nw, "bytes": 1 << (nr + 5 + nw)}
                row["b8"] = measure(c)
                ll.tune("regs_b8", 0)
                row["without_b8"] = measure(c)
                ll.tune("regs_b8", 1)
                rows.append(row)
    ll.tune("regs_shuffle_max_rounds", 4)
    print(json.dumps({"what": __doc__.strip().splitlines()[0], "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
