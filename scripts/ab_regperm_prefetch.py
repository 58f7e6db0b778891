"""Interleaved A/B of the first-wave PDL prefetch (knob regperm_prefetch; pdl_prefetch before session 3's split) on the
register-permutation kernel: register-only pairs of 2^26 elements at every
element width (AUTO = regperm for them), median over rounds."""
import importlib.util
import json
import os
import random
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from scripts.classify_bench import timeit  # noqa: E402
from workloads.values import values_torch  # noqa: E402

spec = importlib.util.spec_from_file_location("tgp", os.path.join(ROOT, "tests", "test_gpu_parity.py"))
tgp = importlib.util.module_from_spec(spec)
spec.loader.exec_module(tgp)


def main():
    for w, r in ((1, 5), (2, 4), (4, 3), (8, 2)):
        c = tgp.perm_pair(random.Random(40 + w), 26, w, r, "reg")
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        n = 1 << A.in_bits
        sets = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                              device="cuda")) for k in range(2)]
        res = {}
        for _ in range(5):
            for pf in (1, 0):
                ll.tune("regperm_prefetch", pf)
                ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path="regperm"))
                res.setdefault("regperm_prefetch=%d" % pf, []).append(2 * n * w / (ms * 1e-3) / 1e9)
        ll.tune("regperm_prefetch", 0)
        print(json.dumps({"elem_bytes": w, "reg_bits": r, "auto_path": ll.plan_describe(A, B, 8 * w)["path"],
                          "gbps_median": {k: round(statistics.median(v)) for k, v in res.items()},
                          "gbps_all": {k: [round(x) for x in v] for k, v in res.items()}}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
