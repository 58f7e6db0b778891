"""Interleaved A/B of every applicable path on the BASELINE configs (one
process, the same buffers; each round times every path once, median over
rounds; CUDA graphs of 50 steps, 2 buffer sets > L2).  GB/s = algorithmic
bytes / time (conversions 2w per element, gathers 2w + 4).

    python scripts/ab_paths.py [rounds] > out.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from scripts.classify_bench import timeit  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import indices_torch, values_torch  # noqa: E402

CONV = ["auto", "smem", "shuffle", "smem_tma", "smem_tma_store", "regperm"]
GATH = ["auto", "shuffle", "smem", "generic"]


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cases = [("cfg2", configs.cfg2()), ("cfg3", configs.cfg3()), ("cfg5", configs.cfg5()),
             ("cfg6", configs.cfg6()), ("cfg4", configs.cfg4()), ("cfg4full", configs.cfg4(variant="full"))]
    for name, c in cases:
        w = c["elem_bytes"]
        res = {}
        if "L" in c:
            L = ll.Layout.from_spec(c["L"])
            n = 1 << L.in_bits
            sets = [(values_torch(n, 4 + k, w, "cuda"), indices_torch(n, 5 + k, c["idx_limit"], "cuda"),
                     torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype, device="cuda")) for k in range(2)]
            nbytes = n * (2 * w + 4)
            paths = []
            for p in GATH:
                try:
                    ll.gather_describe(L, c["axis"], 8 * w, p)
                    paths.append(p)
                except ll.LLError:
                    pass

            def run(p):
                return timeit(lambda i: ll.gather(sets[i % 2][0], sets[i % 2][1], sets[i % 2][2], L, c["axis"],
                                                  8 * w, path=p))
        else:
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            n = 1 << A.in_bits
            sets = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                                      device="cuda")) for k in range(2)]
            nbytes = 2 * n * w
            paths = []
            for p in CONV:
                try:
                    ll.plan_describe(A, B, 8 * w, p)
                    paths.append(p)
                except ll.LLError:
                    pass

            def run(p):
                return timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path=p))
        for _ in range(rounds):
            for p in paths:
                res.setdefault(p, []).append(nbytes / (run(p) * 1e-3) / 1e9)
        auto = (ll.gather_describe(L, c["axis"], 8 * w) if "L" in c else ll.plan_describe(A, B, 8 * w))["path"]
        print(json.dumps({"config": name, "auto_plan": auto,
                          "gbps_median": {p: round(statistics.median(v)) for p, v in res.items()},
                          "gbps_all": {p: [round(x) for x in v] for p, v in res.items()}}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
