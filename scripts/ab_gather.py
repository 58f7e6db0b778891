"""Interleaved A/B of the gather paths x launch-shape knobs (configs 4 and
4full), one process, median over rounds."""
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

VARIANTS = [("auto", {}), ("generic", {}), ("smem", {}), ("smem", {"gather_smem_upc": 0}),
            ("smem", {"gather_smem_upc": 2}), ("smem", {"gather_smem_upc": 4}), ("shuffle", {}),
            ("shuffle", {"gather_shfl_waves": 8}), ("shuffle", {"gather_shfl_waves": 16})]
DEFAULTS = {"gather_smem_upc": 1, "gather_shfl_waves": -1, "gather_pdl": 1, "gather_prefetch_waves": 1}
if len(sys.argv) > 1 and sys.argv[1] == "pdl":   # programmatic dependent launch A/B
    VARIANTS = [(p, kn) for p in ("auto", "generic", "smem", "shuffle") for kn in ({}, {"gather_pdl": 0})]
if len(sys.argv) > 1 and sys.argv[1] == "prefetch":   # smem gather: first-wave bulk prefetch
    VARIANTS = [("smem", kn) for kn in ({}, {"gather_prefetch_waves": 0}, {"gather_prefetch_waves": 2},
                                        {"gather_prefetch_waves": 3})]


def main():
    for name, c in (("cfg4", configs.cfg4()), ("cfg4full", configs.cfg4(variant="full"))):
        w = c["elem_bytes"]
        L = ll.Layout.from_spec(c["L"])
        n = 1 << L.in_bits
        sets = [(values_torch(n, 4 + k, w, "cuda"), indices_torch(n, 5 + k, c["idx_limit"], "cuda"),
                 torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype, device="cuda")) for k in range(2)]
        res = {}
        for _ in range(5 if len(sys.argv) > 1 else 3):
            for p, kn in VARIANTS:
                try:
                    ll.gather_describe(L, c["axis"], 8 * w, p)
                except ll.LLError:
                    continue
                for k, v in kn.items():
                    ll.tune(k, v)
                ms = timeit(lambda i: ll.gather(sets[i % 2][0], sets[i % 2][1], sets[i % 2][2], L, c["axis"],
                                                8 * w, path=p))
                for k in kn:
                    ll.tune(k, DEFAULTS[k])
                res.setdefault(p + " " + json.dumps(kn), []).append(n * (2 * w + 4) / (ms * 1e-3) / 1e9)
        print(json.dumps({"config": name, "gbps_median": {k: round(statistics.median(v)) for k, v in res.items()}}),
              flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
