"""fig:matrix-size on B200: float8 M x N transpose, the
paper's optimal swizzle (LL_PATH_SMEM) against the padding heuristic
(LL_PATH_SMEM_PADDED: unswizzled staging, 16 B pad per 128 B) and an
unswizzled staging buffer.  Graph-replayed timing, GB/s and speedups.

    python scripts/fp8_transpose_sweep.py [--out gpurun_out/fp8_transpose.json]
"""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fp8_transpose.json"))
    ap.add_argument("--sizes", default="10,11,12,13,14")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    bits = [int(x) for x in args.sizes.split(",")]
    res = []
    for mb in bits:
        for nb in bits:
            c = configs.cfg3(n_bits=nb, m_bits=mb)
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            n = 1 << (mb + nb)
            nbytes = 2 * n
            steps = max(20, min(400, (1 << 31) // (nbytes * 4)))
            sets = [(values_torch(n, 3 + s, 1, dev), torch.empty(n, dtype=torch.uint8, device=dev))
                    for s in range(2)]
            row = {"M": 1 << mb, "N": 1 << nb, "bytes": nbytes}
            for path in ("smem", "smem_padded", "smem_noswizzle"):
                try:
                    ms = timeit(lambda i: ll.convert(sets[i % 2][0], A, sets[i % 2][1], B, 8,
                                                     path=path), steps)
                    row[path] = nbytes / ms / 1e6
                except ll.LLError as e:
                    row[path] = None
                    row[path + "_error"] = str(e)
            if row.get("smem") and row.get("smem_padded"):
                row["speedup_vs_padding"] = row["smem"] / row["smem_padded"]
            res.append(row)
            print(json.dumps(row), flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
