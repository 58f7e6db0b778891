"""Interleaved A/B of knob settings on one config's AUTO path (one process,
same buffers, median over rounds; CUDA graphs of 50 steps, 2 buffer sets >
L2).

    python scripts/ab_knobs.py CONFIG 'k=v,k=v;k=v;...' [rounds] > out.jsonl
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
from workloads.values import values_torch  # noqa: E402


# the knobs' defaults (planner.cpp / jit.cpp)
DEFAULTS = {"vec32": 0, "smem_jit_minb": 0, "smem_jit_tpg": 1, "pdl": 1, "smem_jit_single": 0,
            "smem_jit_depth": 1, "run_bytes": 256, "thread_bytes": 64, "tile_order": 0, "auto_asym": 1,
            "ld_hint": 0, "st_hint": 0, "run_bytes_dst": 0, "run_bytes_src": 0, "tmaj_tpc": 2, "pdl_prefetch": 1, "shuffle_pdl": 1, "tile_xor": 0, "tile_xor_skip": 1, "pdl_prefetch_waves": 2, "max_granule": 16, "shuffle_prefetch_waves": 3, "pdl_prefetch_bulk": 1, "shuffle_prefetch_bulk": 1}


def main():
    cfg, sets_spec = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    c = {"2": configs.cfg2, "3": configs.cfg3, "5": configs.cfg5, "6": configs.cfg6}[cfg]()
    w = c["elem_bytes"]
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << A.in_bits
    bufs = [(values_torch(n, 3 + k, w, "cuda"), torch.empty(n, dtype=values_torch(1, 0, w, "cpu").dtype,
                                                              device="cuda")) for k in range(2)]
    variants = [dict(kv.split("=") for kv in s.split(",") if kv) for s in sets_spec.split(";")]
    res = {}
    for _ in range(rounds):
        for v in variants:
            for k, x in v.items():
                ll.tune(k, int(x))
            ms = timeit(lambda i: ll.convert(bufs[i % 2][0], A, bufs[i % 2][1], B, 8 * w))
            for k in v:
                ll.tune(k, DEFAULTS[k])
            res.setdefault(json.dumps(v), []).append(2 * n * w / (ms * 1e-3) / 1e9)
    print(json.dumps({"config": cfg, "gbps_median": {k: round(statistics.median(x)) for k, x in res.items()},
                      "gbps_all": {k: [round(y) for y in x] for k, x in res.items()}}), flush=True)


if __name__ == "__main__":
    main()
