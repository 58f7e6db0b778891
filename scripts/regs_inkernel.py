"""In-kernel cost of one register -> smem -> register conversion on the
register-faithful path (the paper's microbenchmark view: one CTA, the
conversion inside the kernel).  For each case the exchange is
repeated `reps` times inside the kernel; cycles/conversion = (cycles(reps) -
cycles(1)) / (reps - 1), median over trials.  Compares stmatrix/ldmatrix
(regs_matrix=1) against vectorised st/ld.shared only (regs_matrix=0) and,
for warp-local pairs, against the paper's warp-shuffle exchange
in a kernel specialised for the plan (NVRTC).

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


def measure_shuffle(c, reps=256, trials=7):
    """Warp-shuffle exchange (regs_shuffle, NVRTC-specialised): each rep is
    A -> B -> A, so cycles / conversion = delta / (2 (reps - 1))."""
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    plan = ll.plan_describe(A, B, 8 * w, "regs_shuffle")
    n = 1 << A.in_bits
    src = values_torch(n, 3, w, "cuda")
    dst = torch.empty_like(src)
    cy = torch.zeros(1024, dtype=torch.int64, device="cuda")
    per = []
    for _ in range(trials):
        res = []
        for r in (1, reps):
            ll.convert_regs_timed(src, A, dst, B, 8 * w, reps=r, cycles=cy, path="regs_shuffle")
            torch.cuda.synchronize()
            res.append(int(cy[0].item()))
        per.append((res[1] - res[0]) / (2 * (reps - 1)))
    return {"cycles_per_conversion": statistics.median(per), "plan": plan["regs_shuffle"]}


def measure(c, mat, reps=1024, trials=7):
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    ll.tune("regs_matrix", mat)
    ll.tune("regs_shuffle_max_rounds", 0)      # the shared-memory exchange
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
    ll.tune("regs_shuffle_max_rounds", 4)
    return {"cycles_per_conversion": statistics.median(per), "plan": plan["regs"],
            "granule_bytes": plan["granule_bytes"],
            "pred_wavefronts": [plan["pred_wavefronts_per_sts"], plan["pred_wavefronts_per_lds"]]}


def main():
    cases = [("cfg1a Fig.1 A -> mma C (2 warps, fp16)", configs.cfg1("mma")),
             ("cfg1b Fig.1 A -> A^T (2 warps, fp16)", configs.cfg1("T")),
             ("cfg2 one 128x128 tile: mma C -> blocked (4 warps, fp16)", configs.cfg2(batch_bits=0)),
             ("cfg2w one tile, warp-aligned blocked (warp-local: shuffles apply)", configs.cfg2w(batch_bits=0))]
    out = []
    for name, c in cases:
        row = {"case": name}
        for mat in (1, 0):
            row["matrix" if mat else "vector_only"] = measure(c, mat)
        try:
            row["shuffle"] = measure_shuffle(c)
        except ll.LLError as e:
            row["shuffle"] = {"unsupported": str(e)[:120]}
        out.append(row)
    # warp-local pairs of growing register count: the paper's shuffle exchange
    # vs the shared-memory exchange (2^|R| rounds grow with the register bits
    # that change lanes)
    import random
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import rand_warp_local_pair  # noqa: E402
    rng = random.Random(2024)
    sweep = []
    for _ in range(40):
        c = rand_warp_local_pair(rng, 2)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        try:
            sh = measure_shuffle(c, reps=64, trials=3)
        except ll.LLError:
            continue
        sm = measure(c, 1, reps=256, trials=3)
        sweep.append({"reg_bits": c["A"]["in_dims"][0][1], "warps_log2": c["A"]["in_dims"][2][1],
                      "rounds": sh["plan"]["rounds"], "shuffle_cycles": sh["cycles_per_conversion"],
                      "smem_cycles": sm["cycles_per_conversion"], "smem_write": sm["plan"]["write"],
                      "smem_granule_bytes": sm["granule_bytes"]})
        if len(sweep) == 16:
            break
    print(json.dumps({"what": __doc__.strip().splitlines()[0], "sm_clock_note": "cycles = SM clock64",
                      "rows": out, "warp_local_sweep": sweep}, indent=1))


if __name__ == "__main__":
    main()
