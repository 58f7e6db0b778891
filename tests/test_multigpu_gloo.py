"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host path.

The data path has no collective; what the ranks share is the
shard arithmetic and the post-timing reductions.  These run on CPU:

* every rank computes its shard ranges through the C ABI; the all-gathered
  ranges partition both buffers exactly once;
* a rank's destination slice depends only on its source slice: the oracle's
  conversion of a source whose other slices are zeroed reproduces the rank's
  slice of the full conversion;
* max-over-ranks timing and the aggregate GB/s used by bench.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2505_23819_b200 as ll
        from paper_2505_23819_b200 import multigpu
        from oracle import convert as oconv
        from oracle.layout import Layout as OL
        from workloads import configs
        from workloads.values import values_np

        c = configs.cfg5(m_bits=9, kb_bits=8)
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        n = 1 << A.in_bits
        mine = ll.shard_describe(A, B, 8, world, rank)
        allr = multigpu.gather_records(mine)
        ok_partition = multigpu.check_partition([tuple(int(x) for x in r) for r in allr], n, n)
        # independence of the slices (oracle, plain definition)
        Ao, Bo = OL(**c["A"]), OL(**c["B"])
        src = values_np(n, 3, 1)
        full = oconv.convert_np(src, Ao, Bo)
        s0, s1, d0, d1 = mine
        only = np.zeros_like(src)
        only[s0:s1] = src[s0:s1]
        part = oconv.convert_np(only, Ao, Bo)
        ok_slice = bool((part[d0:d1] == full[d0:d1]).all())
        # the other ranks' destination bytes come only from their sources
        outside = np.ones(n, dtype=bool)
        outside[d0:d1] = False
        ok_outside = bool((part[outside] == 0).all())
        objs = multigpu.gather_objects(["%016x" % (rank + 1), rank == 0])
        assert objs == [["%016x" % 1, True], ["%016x" % 2, False]]
        t = multigpu.max_over_ranks(10.0 + rank)
        agg = multigpu.aggregate_gbps([2 * (s1 - s0)] * world, [10.0, 11.0], "strong")
        q.put((rank, ok_partition, ok_slice, ok_outside, t, agg))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, "error", repr(e)))


def test_two_rank_gloo_shards():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
        rank, ok_partition, ok_slice, ok_outside, t, agg = r
        assert ok_partition and ok_slice and ok_outside
        assert t == 11.0                                    # max over ranks
        n = 1 << 17
        assert abs(agg - (2 * n) / (11.0e-3) / 1e9) < 1e-9   # all bytes / slowest rank


def test_aggregate_single_process():
    from paper_2505_23819_b200 import multigpu
    assert multigpu.max_over_ranks(3.5) == 3.5
    assert multigpu.gather_records([1, 2]) == [[1, 2]]
    assert multigpu.gather_objects(["ab", None]) == [["ab", None]]
    with pytest.raises(ValueError):
        multigpu.aggregate_gbps([1], [1.0], "sideways")
