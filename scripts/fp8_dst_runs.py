"""fp8 transposes: destination coalescing run length (knob run_bytes_dst)
vs the planner's default (asymmetric 64 B when the group would be >= 4 warps).
python scripts/fp8_dst_runs.py > out.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from sweep import timeit  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402

dev = torch.device("cuda", 0)
res = []
for mb, nb in ((13, 13), (14, 14), (12, 14), (14, 12)):
    c = configs.cfg3(n_bits=nb, m_bits=mb)
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    n = 1 << (mb + nb)
    sets = [(values_torch(n, 3 + s, 1, dev), torch.empty(n, dtype=torch.uint8, device=dev)) for s in range(2)]
    for rd in (0, 32, 16):
        ll.tune("run_bytes_dst", rd)
        g = ll.plan_describe(A, B, 8, "smem")["group_warps_log2"]
        ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8), 100)
        res.append({"M": 1 << mb, "N": 1 << nb, "run_bytes_dst": rd, "group_warps_log2": g,
                    "GBps": 2 * n / ms / 1e6})
        print(json.dumps(res[-1]), flush=True)
ll.tune("run_bytes_dst", 0)
