"""Bandwidth ceilings for write-heavy traffic (the mxfp4 upcast reads 1 byte
and writes 4): torch write-only fill, 1:4 broadcast copy, 1:1 copy.
Graph-replayed, 2 rotating buffer sets > L2.  Writes gpurun_out/write_ceiling.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from scripts.sweep import timeit  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 29
src = [torch.randint(0, 255, (n,), dtype=torch.uint8, device=dev) for _ in range(2)]
dst = [torch.empty(4 * n, dtype=torch.uint8, device=dev) for _ in range(2)]
res = []


def emit(name, ms, nbytes):
    r = {"case": name, "ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1)}
    res.append(r)
    print(json.dumps(r), flush=True)


emit("write_only_fill 2GiB", timeit(lambda i: dst[i % 2].fill_(i & 0xFF), 50), 4 * n)
emit("read1_write4 broadcast", timeit(lambda i: dst[i % 2].view(n, 4).copy_(src[i % 2].view(n, 1).expand(n, 4)), 50), 5 * n)
emit("copy 1:1 512MiB", timeit(lambda i: dst[i % 2][:n].copy_(src[i % 2]), 50), 2 * n)
emit("copy 1:1 2GiB", timeit(lambda i: dst[i % 2].copy_(dst[1 - i % 2]), 20), 8 * n)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "write_ceiling.json"), "w"), indent=1)
