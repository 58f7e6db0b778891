"""Sweep ll_convert_host chunking (host_chunk_mb x host_slots) on cfg2 / cfg5,
plus raw pinned-copy bandwidth for context.  Writes gpurun_out/e2e_sweep.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = []
for cfg in ("2", "5"):
    if cfg == "2":
        c = configs.cfg2(batch_bits=0)
        nb, n = 1 << 12, 1 << 26
    else:
        c = configs.cfg5()
        nb, n = 1, 1 << 29
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    w = c["elem_bytes"]
    src = values_torch(n, 9, w, "cpu").pin_memory()
    dst = torch.empty_like(src).pin_memory()
    for mb in (2, 4, 8, 16):
        for slots in (2, 3, 4):
            ll.tune("host_chunk_mb", mb)
            ll.tune("host_slots", slots)
            scratch = slots * mb << 20
            ds = torch.empty(scratch, dtype=torch.uint8, device="cuda")
            dd = torch.empty(scratch, dtype=torch.uint8, device="cuda")
            ms = timed(lambda: ll.convert_host(src, A, dst, B, 8 * w, nb, ds, dd, scratch))
            r = {"cfg": cfg, "chunk_mb": mb, "slots": slots, "ms": round(ms, 3),
                 "GBps": round(2 * n * w / ms / 1e6, 1)}
            res.append(r)
            print(json.dumps(r), flush=True)
            del ds, dd
x = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()
h2 = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()
x2 = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()


def both():
    x.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(x2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


for name, fn, nbytes in (("h2d", lambda: x.copy_(h, non_blocking=True), 1 << 28),
                         ("d2h", lambda: h.copy_(x, non_blocking=True), 1 << 28),
                         ("h2d+d2h concurrent", both, 2 << 28)):
    ms = timed(fn)
    r = {"copy": name, "GBps": round(nbytes / ms / 1e6, 1)}
    res.append(r)
    print(json.dumps(r), flush=True)
# host-side enqueue cost of one conversion launch (no sync inside the loop)
import time  # noqa: E402
c = configs.cfg2(batch_bits=0)
A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
xs = torch.zeros(1 << 14, dtype=torch.int16, device="cuda")
xd = torch.empty_like(xs)
for _ in range(100):
    ll.convert(xs, A, xd, B, 16)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    ll.convert(xs, A, xd, B, 16)
t1 = time.perf_counter()
torch.cuda.synchronize()
r = {"host_enqueue_us_per_convert": round((t1 - t0) / 2000 * 1e6, 2)}
res.append(r)
print(json.dumps(r), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "e2e_sweep.json"), "w"), indent=1)
