"""The global-access pattern's own ceiling per config: the compiled smem
kernel with the shared-memory exchange removed (knob smem_jit_noxchg: the
identical loads and stores, data left in place -- wrong output, same DRAM
pattern) vs the real conversion vs a flat device copy of the same bytes
(torch copy_ / cudaMemcpy D2D), interleaved, median of rounds."""
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
    for name, c in (("cfg2", configs.cfg2()), ("cfg3", configs.cfg3()), ("cfg5", configs.cfg5()),
                    ("cfg6", configs.cfg6())):
        w = c["elem_bytes"]
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        n = 1 << A.in_bits
        sets = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                                  device="cuda")) for k in range(2)]
        res = {}
        for _ in range(3):
            for tag in ("smem", "smem_noxchg", "copy"):
                if tag == "copy":
                    ms = timeit(lambda i: sets[i % 2][1].copy_(sets[i % 2][0]))
                else:
                    ll.tune("smem_jit_noxchg", 1 if tag == "smem_noxchg" else 0)
                    ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path="smem"))
                    ll.tune("smem_jit_noxchg", 0)
                res.setdefault(tag, []).append(2 * n * w / (ms * 1e-3) / 1e9)
        print(json.dumps({"config": name, "gbps_median": {k: round(statistics.median(v)) for k, v in res.items()},
                          "gbps_all": {k: [round(x) for x in v] for k, v in res.items()}}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
