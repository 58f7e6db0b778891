"""Interleaved A/B of programmatic dependent launch on the compiled mxfp4
upcast (knob upcast_pdl), config 5 at full size, median over rounds."""
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


def main():
    c = configs.cfg5()
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    sc = (indices_torch(n // 16, 42, 16, "cuda") + 120).to(torch.uint8)
    sets = [(values_torch(n, 3 + k, 1, "cuda"), torch.empty(2 * n, dtype=torch.int16, device="cuda"))
            for k in range(2)]
    nbytes = n + n // 16 + 4 * n
    res = {}
    for _ in range(5):
        for pdl in (0, 1):
            ll.tune("upcast_pdl", pdl)
            ms = timeit(lambda i: ll.mxfp4_upcast(sets[i % 2][0], A, sc, sets[i % 2][1], B), steps=20)
            res.setdefault("upcast_pdl=%d" % pdl, []).append(nbytes / (ms * 1e-3) / 1e9)
    ll.tune("upcast_pdl", 0)
    print(json.dumps({"config": "cfg5 upcast", "gbps_median": {k: round(statistics.median(v)) for k, v in res.items()},
                      "gbps_all": {k: [round(x) for x in v] for k, v in res.items()}}), flush=True)


if __name__ == "__main__":
    main()
