"""Register-permutation kernel (LL_PATH_REGPERM) launch / access variants vs
the smem and shuffle paths on register-only pairs (2^26 elements, CUDA-graph
timing as scripts/classify_bench.py)."""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from scripts.classify_bench import timeit  # noqa: E402
from tests.test_gpu_parity import perm_pair  # noqa: E402
from workloads.values import values_torch  # noqa: E402

VARIANTS = [{}, {"regperm_occ": 2}, {"regperm_occ": 3}, {"regperm_occ": 4}, {"regperm_occ": 6},
            {"regperm_u": 2}, {"regperm_u": 8}, {"regperm_occ": 4, "regperm_u": 2}]


def main():
    d = 26
    for w, r in ((4, 3), (4, 2), (2, 3), (1, 4), (1, 5)):
        rng = random.Random(7 + w)
        c = perm_pair(rng, d, w, r, "reg")
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        n = 1 << d
        sets = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                                  device="cuda")) for k in range(2)]
        row = {"w": w, "reg_bits": r}
        for path in ("smem", "shuffle"):
            ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path=path))
            row[path] = round(2 * n * w / (ms * 1e-3) / 1e9)
        for v in VARIANTS:
            for k, x in v.items():
                ll.tune(k, x)
            ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path="regperm"))
            row["regperm " + json.dumps(v)] = round(2 * n * w / (ms * 1e-3) / 1e9)
            for k in v:
                ll.tune(k, {"pdl": 1, "regperm_waves": 0, "regperm_v8": -1, "regperm_occ": 0}.get(k, 0))
        print(json.dumps(row), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
