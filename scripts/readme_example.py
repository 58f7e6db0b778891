"""The README usage snippet, runnable (GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch, paper_2505_23819_b200 as ll
from workloads import configs

c = configs.cfg2()                                   # mma C fragment -> blocked, 4096 tiles
A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
src = torch.empty(1 << A.in_bits, dtype=torch.int16, device="cuda")
dst = torch.empty_like(src)
ll.convert(src, A, dst, B, 16)                       # planner's choice (AUTO)
ll.convert(src, A, dst, B, 16, path="smem_tma")      # or a specific path
print(ll.plan_describe(A, B, 16))                    # the plan as JSON
