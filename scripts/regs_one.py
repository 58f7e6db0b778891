"""One timed register-faithful launch (for ncu): python scripts/regs_one.py CFG MODE REPS
MODE: 1 / 0 = shared-memory exchange with / without stmatrix-ldmatrix,
"shfl" = the NVRTC-specialised warp-shuffle exchange (warp-local pairs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402

cfg, mode, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
c = {"1a": lambda: configs.cfg1("mma"), "1b": lambda: configs.cfg1("T"),
     "2": lambda: configs.cfg2(batch_bits=0), "2w": lambda: configs.cfg2w(batch_bits=0)}[cfg]()
w = c["elem_bytes"]
A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
path = "regs_shuffle" if mode == "shfl" else "regs"
if mode != "shfl":
    ll.tune("regs_matrix", int(mode))
    ll.tune("regs_shuffle_max_rounds", 0)
src = values_torch(1 << A.in_bits, 3, w, "cuda")
dst = torch.empty_like(src)
cy = torch.zeros(16, dtype=torch.int64, device="cuda")
ll.convert_regs_timed(src, A, dst, B, 8 * w, reps=reps, cycles=cy, path=path)
torch.cuda.synchronize()
print(cfg, mode, reps, int(cy[0].item()))
