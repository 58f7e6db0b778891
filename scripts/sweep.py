"""Tuning / ablation sweep on one GPU: GB/s per (config, path, knobs), plus a
torch copy_ of the same number of bytes as the practical ceiling.

    python scripts/sweep.py [--configs 2,3,4,5] [--steps 100] [--out gpurun_out/sweep.json]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import indices_torch, values_torch  # noqa: E402


DEFAULTS = {"tpg": 2, "pipe": 1, "carveout": -1, "pow2": 0, "stages": 3, "async_tpg": 8, "thread_bytes": 64,
            "thread_bytes_max": 128, "max_granule": 16, "run_bytes": 256, "tile_order": 0}


def timeit(step, steps, warm=5):
    """Average ms per step: `steps` steps captured in a CUDA graph, replayed."""
    for i in range(warm):
        step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            for i in range(steps):
                step(i)
    torch.cuda.current_stream().wait_stream(cap)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--knobs", default="tpg=0,1,2,4,8;pipe=0,1")
    ap.add_argument("--paths", default="smem,smem_noswizzle,generic")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = []

    def emit(r):
        res.append(r)
        print(json.dumps(r), flush=True)

    knob_sets = [{}]
    for part in args.knobs.split(";"):
        if not part:
            continue
        name, vals = part.split("=")
        knob_sets = [dict(k, **{name: int(v)}) for k in knob_sets for v in vals.split(",")]

    for cfg in args.configs.split(","):
        if cfg == "4":
            c = configs.cfg4()
            L = ll.Layout.from_spec(c["L"])
            n = 1 << L.in_bits
            nbytes = n * 12
            sets = [(values_torch(n, 4 + s, 4, dev), indices_torch(n, 5 + s, 32, dev),
                     torch.empty(n, dtype=torch.int32, device=dev)) for s in range(3)]
            for path in ("shuffle", "generic"):
                for vpt in (1, 2, 4, 8):
                    ll.tune("gather_vpt", vpt)
                    ms = timeit(lambda i: ll.gather(*sets[i % 3][:3], L, 2, 32, path=path),
                                args.steps)
                    emit({"cfg": cfg, "path": path, "gather_vpt": vpt, "ms": ms,
                          "GBps": nbytes / ms / 1e6})
            ll.tune("gather_vpt", 2)
            a = [torch.empty(nbytes // 2, dtype=torch.uint8, device=dev) for _ in range(3)]
            b = [torch.empty(nbytes // 2, dtype=torch.uint8, device=dev) for _ in range(3)]
        else:
            c = {"2": configs.cfg2, "3": configs.cfg3, "5": configs.cfg5, "1": configs.cfg1}[cfg]()
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            w = c["elem_bytes"]
            n = 1 << A.in_bits
            nbytes = 2 * n * w
            nsets = 2 if n * w >= (64 << 20) else 4
            sets = [(values_torch(n, 7 + s, w, dev), values_torch(n, 0, w, dev)) for s in range(nsets)]
            if "upcast" in args.paths.split(",") and cfg == "5":
                # fused mxfp4 -> bf16 (2 bf16 per packed byte), scales in [120, 135]
                scales = (indices_torch(n // 16, 42, 16, dev) + 120).to(torch.uint8)
                usets = [(sets[s][0], torch.empty(2 * n, dtype=torch.int16, device=dev))
                         for s in range(nsets)]
                for ks in knob_sets:
                    for k, v in ks.items():
                        ll.tune(k, v)
                    try:
                        ms = timeit(lambda i: ll.mxfp4_upcast(usets[i % nsets][0], A, scales,
                                                              usets[i % nsets][1], B), args.steps)
                        emit(dict({"cfg": cfg, "path": "upcast", "ms": ms,
                                   "GBps": (n + n // 16 + 4 * n) / ms / 1e6}, **ks))
                    except ll.LLError as e:
                        emit(dict({"cfg": cfg, "path": "upcast", "error": str(e)}, **ks))
                    for k, v in DEFAULTS.items():
                        ll.tune(k, v)
                del usets
            for path in [q for q in args.paths.split(",") if q != "upcast"]:
                for ks in (knob_sets if path.startswith("smem") or path == "shuffle" else [{}]):
                    for k, v in ks.items():
                        ll.tune(k, v)
                    try:
                        ms = timeit(lambda i: ll.convert(sets[i % nsets][0], A, sets[i % nsets][1],
                                                         B, 8 * w, path=path), args.steps)
                        emit(dict({"cfg": cfg, "path": path, "ms": ms, "GBps": nbytes / ms / 1e6},
                                  **ks))
                    except ll.LLError as e:
                        emit({"cfg": cfg, "path": path, "error": str(e)})
                    for k, v in DEFAULTS.items():
                        ll.tune(k, v)
            a = [torch.empty(nbytes // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
            b = [torch.empty(nbytes // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
        ms = timeit(lambda i: b[i % len(b)].copy_(a[i % len(a)]), args.steps)
        emit({"cfg": cfg, "path": "torch_copy_same_bytes", "ms": ms, "GBps": nbytes / ms / 1e6})
        if cfg == "3":
            m = 1 << 13
            ta = [values_torch(m * m, 3 + s, 2, dev).view(m, m) for s in range(2)]
            tb = [torch.empty(m, m, dtype=torch.int16, device=dev) for _ in range(2)]
            ms = timeit(lambda i: tb[i % 2].copy_(ta[i % 2].t()), args.steps)
            emit({"cfg": cfg, "path": "torch_transpose_copy", "ms": ms, "GBps": nbytes / ms / 1e6})
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
