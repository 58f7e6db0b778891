"""Multi-GPU plumbing around the C ABI (one process per GPU, torch.distributed).

The conversion partitions into independent tiles, so there is no collective
on the data path:

* weak scaling: every rank converts its own full batch;
* strong scaling: rank r converts shard r of the top block bits
  (``ll_convert_shard``), holding only its slices of src and dst.

The only cross-rank traffic is after the timed region: the max of the
per-rank times (and optionally per-rank checksums) with one all-reduce /
all-gather.  These helpers are plain host logic, covered by gloo tests on CPU.
"""

import torch
import torch.distributed as dist

from . import _lib


def shard_slices(A, B, elem_bits, world, path="auto"):
    """Byte ranges [(src_begin, src_end, dst_begin, dst_end)] of every rank."""
    return [_lib.shard_describe(A, B, elem_bits, world, r, path) for r in range(world)]


def check_partition(slices, src_bytes, dst_bytes):
    """True iff the slices tile both buffers exactly once, in rank order."""
    s = sorted(slices)
    if s[0][0] != 0 or s[-1][1] != src_bytes:
        return False
    d = sorted((x[2], x[3]) for x in slices)
    if d[0][0] != 0 or d[-1][1] != dst_bytes:
        return False
    for a, b in zip(s, s[1:]):
        if a[1] != b[0]:
            return False
    for a, b in zip(d, d[1:]):
        if a[1] != b[0]:
            return False
    return True


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (identity without a process group)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_records(record, device=None):
    """All-gather a small list of floats per rank (e.g. checksum, time)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [list(record)]
    t = torch.tensor([float(x) for x in record], dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def gather_objects(obj):
    """All-gather one picklable record per rank (e.g. checksum strings)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def aggregate_gbps(bytes_per_rank, time_ms_per_rank, scaling):
    """Whole-job GB/s: all ranks' bytes / the slowest rank's time.

    ``bytes_per_rank``: list (one per rank) of algorithmic bytes each rank moved.
    ``time_ms_per_rank``: list of each rank's device time for the same region."""
    if scaling not in ("weak", "strong"):
        raise ValueError("scaling must be weak or strong")
    t = max(time_ms_per_rank)
    return sum(bytes_per_rank) / (t * 1e-3) / 1e9
