"""Per-rank work of config 5's strong scaling, measured on ONE GPU: the
shard a rank owns at N = 1, 2, 4, 8 (ll_convert_shard of shard 0, its own
slices, 2 rotating buffer sets, CUDA graphs) -> GB/s per rank and N x that
as the aggregate the N-GPU run would reach if the ranks do not interfere
(no collective on the hot path).  A projection, not a
multi-GPU measurement: it prices the shrinking per-rank launch (launch
latency, tail wave) that strong scaling exposes."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_23819_b200 as ll  # noqa: E402
from workloads import configs  # noqa: E402
from workloads.values import values_torch  # noqa: E402


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
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / steps)
    return statistics.median(out)


def main():
    # optional knobs: python scripts/shard_projection.py k=v,k=v
    for kv in (sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] else []):
        k, v = kv.split("=")
        ll.tune(k, int(v))
    c = configs.cfg5()
    A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
    total = 2 << A.in_bits   # bytes moved by the whole job (1 B read + 1 B written per element)
    src = values_torch(1 << A.in_bits, 6, 1, "cuda")
    rows = []
    for n in (1, 2, 4, 8):
        s0, s1, d0, d1 = ll.shard_describe(A, B, 8, n, 0)
        sets = [(src.view(torch.uint8)[s0:s1].clone(), torch.empty(d1 - d0, dtype=torch.uint8, device="cuda"))
                for _ in range(2)]
        ms = timeit(lambda i: ll.convert_shard(sets[i % 2][0], A, sets[i % 2][1], B, 8, n, 0))
        per_rank = (total // n) / (ms * 1e-3) / 1e9
        rows.append({"n_gpus": n, "shard_bytes_moved": total // n, "ms_per_step": round(ms, 5),
                     "gbps_per_rank": round(per_rank), "projected_aggregate_gbps": round(per_rank * n)})
        print(json.dumps(rows[-1]), flush=True)
        del sets
        torch.cuda.empty_cache()
    base = rows[0]["projected_aggregate_gbps"]
    print(json.dumps({"projected_speedup_8_over_1": round(rows[-1]["projected_aggregate_gbps"] / base, 2)}))


if __name__ == "__main__":
    main()
