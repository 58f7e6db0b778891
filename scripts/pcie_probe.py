"""PCIe ceiling for the end-to-end numbers: pinned host <-> device copies of
512 MiB, H2D alone, D2H alone and both at once on two streams (what
ll_convert_host overlaps), CUDA events, best of 5."""
import json
import torch

n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    best = None
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


res = {}
ms = timed(lambda: d_in.copy_(h_in, non_blocking=True))
res["h2d_GBps"] = round(n / ms / 1e6, 1)
ms = timed(lambda: h_out.copy_(d_out, non_blocking=True))
res["d2h_GBps"] = round(n / ms / 1e6, 1)
ms = timed(both)
res["both_directions_total_GBps"] = round(2 * n / ms / 1e6, 1)
res["bytes_each_way"] = n
print(json.dumps(res))
