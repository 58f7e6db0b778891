"""Row-major -> column-major transposes of 2^28 bytes at every element width
(config 3's layout family): which part of config 3's gap to the copy figure
comes from the access pattern and which from the exchange (sub-word prmt,
8 vectors per thread).  Interleaved A/B of the smem / TMA paths."""
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
from workloads.values import values_torch  # noqa: E402


def main():
    for w, m, n in ((1, 14, 14), (2, 13, 13), (4, 13, 12), (8, 12, 12), (2, 12, 14), (2, 14, 12)):
        c = configs.cfg3(n_bits=n, m_bits=m)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        N = 1 << (m + n)
        sets = [(values_torch(N, 3 + k, w, "cuda"), torch.empty(N, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                                  device="cuda")) for k in range(2)]
        res = {}
        paths = []
        for p in ("smem", "smem_tma", "smem_tma_store"):
            try:
                ll.plan_describe(A, B, 8 * w, p)
                paths.append(p)
            except ll.LLError:
                pass
        for _ in range(3):
            for p in paths:
                ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path=p))
                res.setdefault(p, []).append(2 * N * w / (ms * 1e-3) / 1e9)
        d = ll.plan_describe(A, B, 8 * w)
        print(json.dumps({"elem_bytes": w, "rows_log2": m, "cols_log2": n,
                          "plan": {k: d.get(k) for k in ("granule_bytes", "vectors_per_thread", "group_warps_log2", "swaps")},
                          "gbps_median": {p: round(statistics.median(v)) for p, v in res.items()}}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
