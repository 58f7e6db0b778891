"""AUTO's HBM-path classification, measured (register permutation
/ warp shuffles / shared memory).

Pairs of distributed layouts over 2^26 elements that differ only in register
order (no exchange between threads) or only in lane order (warp-local), at
each element width; every applicable path timed with CUDA events over CUDA
graph replays (2 buffer sets > L2), GB/s = 2 x bytes / time.

    python scripts/classify_bench.py > out.json
"""

import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_2505_23819_b200 as ll
from tests.test_gpu_parity import perm_pair
from workloads.values import values_torch


def timeit(fn, steps=50, reps=5):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        best = ms if best is None else min(best, ms)
    return best


def main():
    d = 26
    res = []
    for w in (1, 2, 4, 8):
        vb = {1: 4, 2: 3, 4: 2, 8: 1}[w]
        rng = random.Random(7 + w)
        for which, r in (("reg", vb), ("reg", vb + 1), ("reg", vb + 2), ("lane", vb)):
            if which == "reg" and r < 2:
                continue          # a single register bit has no permutation
            c = perm_pair(rng, d, w, r, which)
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            n = 1 << d
            sets = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                                      device="cuda")) for k in range(2)]
            row = {"w": w, "differs_in": which, "reg_bits": r, "bytes": 2 * n * w,
                   "auto": ll.plan_describe(A, B, 8 * w)["path"]}
            for path in ("auto", "regperm", "shuffle", "smem"):
                try:
                    ll.plan_describe(A, B, 8 * w, path)
                except ll.LLError:
                    continue
                ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8 * w, path=path))
                row[path + "_gbps"] = 2 * n * w / (ms * 1e-3) / 1e9
            res.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
            del sets
            torch.cuda.empty_cache()
    print(json.dumps({"rows": res}, indent=1))


if __name__ == "__main__":
    main()
