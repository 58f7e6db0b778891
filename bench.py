"""Benchmark of the hot path: layout conversion (and gather) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Default workload = BASELINE.json configs[1] ("cfg2"): mma.sync m16n8k16
accumulator layout -> coalesced blocked layout, 128x128 fp16 tiles, batch
4096 (2^26 elements, 128 MiB in + 128 MiB out).  One step = one ll_convert
over the whole batch (planning is cached on the host; the kernel does the
rest).  Inputs are synthetic (seeded splitmix64 patterns, generated on the
device).  Timing: W untimed warm-up steps, then K steps bracketed by a barrier
and torch.cuda.synchronize(), CUDA events on the launching stream; buffer
sets rotate so the footprint (>= 4 x 128 MiB) exceeds the 126 MB L2.
Multi-GPU: one process per GPU (torchrun), each rank converts its own batch
(weak scaling, no collective on the hot path); time = max over ranks.

Prints ONE JSON line (rank 0).
"""

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "convert_layout effective GB/s vs 8 TB/s HBM peak; smem bank conflicts/request"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="2", choices=["1", "2", "3", "4", "5"])
    ap.add_argument("--path", default="auto")
    ap.add_argument("--upcast", action="store_true",
                    help="config 5 only: fused mxfp4 dequantisation to bf16 (NEXT #1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank converts the full workload; strong: rank r converts "
                         "shard r of the top block bits (ll_convert_shard, cfg2/cfg5)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tune", action="append", default=[], metavar="KNOB=VALUE",
                    help="ll_tune knob before planning (e.g. tma_stages=4); repeatable")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch each step from Python instead of replaying a CUDA graph")
    return ap.parse_args()


# ----------------------------------------------------------------- workloads

def workload(cfg):
    from workloads import configs
    if cfg == "1":
        c = configs.cfg1("mma")
        desc = "cfg1: paper Fig.1 16x16 fp16, 2 warps, layout A -> B (mma C fragment, reading A3)"
    elif cfg == "2":
        c = configs.cfg2()
        desc = ("cfg2: mma.sync m16n8k16 accumulator -> blocked [1,8]x[2,16]x[4,1], "
                "128x128 fp16 tiles, batch 4096")
    elif cfg == "3":
        c = configs.cfg3()
        desc = "cfg3: row-major -> column-major transpose, 8192x8192 bf16"
    elif cfg == "4":
        c = configs.cfg4()
        desc = "cfg4: tl.gather along the 32-wide axis of [4096,128,32] fp32, int32 idx (reading A21)"
    else:
        c = configs.cfg5()
        desc = "cfg5: mxfp4 packed [32768,16384] u8, blocked -> packed mma A-fragment (reading A22)"
    return c, desc


def algorithmic_bytes(cfg, c):
    from workloads.configs import total_elems
    if cfg == "4":
        n = total_elems(c["L"])
        return n * c["elem_bytes"] * 2 + n * 4
    return total_elems(c["A"]) * c["elem_bytes"] + total_elems(c["B"]) * c["elem_bytes"]


# ------------------------------------------------------------------- clocks

class ClockSampler:
    """NVML polling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index=0, period=0.001):
        self.period = period
        self.samples = []
        self.reasons = set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ----------------------------------------------------------------- helpers

def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary; cfg is the key ("2", "5_upcast", "3_tma", "2_regs", ...)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("cfg" + cfg, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_baseline(cfg, c, budget_s=12.0):
    """The oracle as it stands (oracle.convert.convert_np / gather_np, the
    plain definition), single process, on a bounded sample of the workload:
    a prefix of the batch (whole layout instances), scaled to GB/s."""
    import numpy as np
    from oracle import convert as oconv
    from oracle.layout import Layout as OL
    from workloads import configs
    from workloads.values import indices_np, values_np
    t0 = time.time()
    if cfg == "2":
        # sample: batch of 2^k tiles of the same layout family
        k = 4
        cs = configs.cfg2(batch_bits=k)
        A, B = OL(**cs["A"]), OL(**cs["B"])
        n = 1 << A.in_bits
        src = values_np(n, 7, 2)
        reps = 0
        t0 = time.time()
        while True:
            oconv.convert_np(src, A, B)
            reps += 1
            if time.time() - t0 > budget_s:
                break
        dt = time.time() - t0
        nbytes = reps * n * 2 * 2
        sample = "%d x convert_np on cfg2 with 2^%d tiles (%d elements)" % (reps, k, n)
    elif cfg == "4":
        cs = configs.cfg4(r_bits=6)
        L = OL(**cs["L"])
        n = 1 << L.in_bits
        src = values_np(n, 4, 4)
        idx = indices_np(n, 5, 32)
        reps = 0
        t0 = time.time()
        while True:
            oconv.gather_np(src, idx, L, 2)
            reps += 1
            if time.time() - t0 > budget_s:
                break
        dt = time.time() - t0
        nbytes = reps * n * 12
        sample = "%d x gather_np on [64,128,32] fp32" % reps
    else:
        if cfg == "3":
            cs = configs.cfg3(n_bits=10)
        elif cfg == "5":
            cs = configs.cfg5(m_bits=11, kb_bits=10)
        else:
            cs = configs.cfg1("mma")
        A, B = OL(**cs["A"]), OL(**cs["B"])
        n = 1 << A.in_bits
        w = cs["elem_bytes"]
        src = values_np(n, 7, w)
        reps = 0
        t0 = time.time()
        while True:
            oconv.convert_np(src, A, B)
            reps += 1
            if time.time() - t0 > budget_s:
                break
        dt = time.time() - t0
        nbytes = reps * n * w * 2
        sample = "%d x convert_np on %s (%d elements)" % (reps, cs.get("name"), n)
    return {"value": nbytes / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": sample, "host_cpus": os.cpu_count(), "seconds": round(dt, 2)}


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    c, desc = workload(cfg)
    steps = []
    for _ in range(args.warmup):
        pass
    budget = max(1.0, 90.0 / max(1, args.steps))
    vals = []
    for _ in range(max(1, args.steps)):
        b = cpu_baseline(cfg, c, budget_s=budget)
        vals.append(b)
    v = sum(x["value"] for x in vals) / len(vals)
    b0 = vals[0]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(x["seconds"] for x in vals) * 1000 / len(vals),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic", "config": {"workload": desc, "sample": b0["sample"]},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": b0["sample"], "host_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_2505_23819_b200 as ll
    from workloads.values import indices_torch, values_torch
    for kv in args.tune:
        k, v = kv.split("=")
        ll.tune(k, int(v))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg = args.config
    c, desc = workload(cfg)
    nbytes = algorithmic_bytes(cfg, c)
    stream = torch.cuda.current_stream()

    if cfg == "4":
        L = ll.Layout.from_spec(c["L"])
        n = 1 << L.in_bits
        sets = [(values_torch(n, 4 + s + 10 * rank, 4, dev), indices_torch(n, 5 + s, 32, dev),
                 torch.empty(n, dtype=torch.int32, device=dev)) for s in range(2)]

        def step(i):
            s, ix, o = sets[i % 2]
            ll.gather(s, ix, o, L, c["axis"], 32, path=args.path)
        plan = ll.gather_describe(L, c["axis"], 32, args.path)
    else:
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        w = c["elem_bytes"]
        n = 1 << A.in_bits
        if args.scaling == "strong" and world > 1:
            # this rank holds and converts only its shard (contiguous slices)
            s0, s1, d0, d1 = ll.shard_describe(A, B, 8 * w, world, rank, args.path)
            n_loc = (s1 - s0) // w
            nbytes = (s1 - s0) + (d1 - d0)
        else:
            n_loc = n
        nsets = max(2, -(-(2 * 128 << 20) // (2 * n_loc * w)) + 1) if n_loc * w < (128 << 20) else 2
        nsets = min(nsets, 64)
        sets = [(values_torch(n_loc, 7 + s + 10 * rank, w, dev),
                 torch.empty(n_loc, dtype=values_torch(1, 0, w, "cpu").dtype, device=dev))
                for s in range(nsets)]

        if args.upcast:
            # fused mxfp4 -> bf16: 2 bf16 per packed byte, scales [M][K/32]
            n_sc = n // 16
            scales = (indices_torch(n_sc, 42, 16, dev) + 120).to(torch.uint8)
            sets = [(s_, torch.empty(2 * n_loc, dtype=torch.int16, device=dev)) for s_, _ in sets]
            nbytes = n * w + n_sc + 4 * n * w

        def step(i):
            s, d = sets[i % len(sets)]
            if args.upcast:
                ll.mxfp4_upcast(s, A, scales, d, B)
                return
            if args.scaling == "strong" and world > 1:
                ll.convert_shard(s, A, d, B, 8 * w, world, rank, path=args.path)
            else:
                ll.convert(s, A, d, B, 8 * w, path=args.path)
        plan = ll.plan_describe(A, B, 8 * w, args.path)

    torch.cuda.synchronize()
    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    K = args.steps
    graph = None
    l0 = ll.launch_count()
    if not args.no_graph:
        # the K steps are captured once into a CUDA graph (the library launches
        # on the capturing stream) and replayed: no host launch gaps in the region
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                for i in range(K):
                    step(i)
        torch.cuda.current_stream().wait_stream(cap)
        launches = ll.launch_count() - l0
        graph.replay()                      # warm the graph itself
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(K):
                step(i)
        e1.record(stream)
        torch.cuda.synchronize()
    if graph is None:
        launches = ll.launch_count() - l0
    total_ms = e0.elapsed_time(e1)
    from paper_2505_23819_b200 import multigpu
    if world > 1:
        dist.barrier()
    total_ms = multigpu.max_over_ranks(total_ms, device=dev)
    ms_per_step = total_ms / K
    value = multigpu.aggregate_gbps([nbytes] * world, [ms_per_step] * world, args.scaling)
    avg_launch_ms = total_ms / K
    achieved = nbytes / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    from paper_2505_23819_b200 import multigpu
    # row a12 (untimed): checksum record of the last step's destination per
    # rank (ll_checksum, indexed), and for conversions the permutation
    # property on the whole buffer (index-free checksums of src and dst agree)
    last = sets[(K - 1) % len(sets)]
    dst_t = last[2] if cfg == "4" else last[1]
    ck = torch.zeros(3, dtype=torch.int64, device=dev)
    ll.checksum(dst_t, dst_t.numel(), 8 * dst_t.element_size(), ck[0:1], stream=stream)
    perm_check = cfg != "4" and not args.upcast
    if perm_check:
        ll.checksum(last[0], last[0].numel(), 8 * last[0].element_size(), ck[1:2], indexed=False,
                    stream=stream)
        ll.checksum(dst_t, dst_t.numel(), 8 * dst_t.element_size(), ck[2:3], indexed=False,
                    stream=stream)
    torch.cuda.synchronize()
    ckv = [int(x) & ((1 << 64) - 1) for x in ck.cpu().tolist()]
    records = multigpu.gather_objects(["%016x" % ckv[0], (ckv[1] == ckv[2]) if perm_check else None])
    verify = {"dst_checksum_per_rank": [r[0] for r in records],
              "permutation_ok": all(r[1] for r in records) if perm_check else None,
              "how": "ll_checksum (row a12): indexed splitmix64 sum of the last step's destination; "
                     "permutation_ok = index-free sums of src and dst agree"}

    # end to end through the C ABI with HOST buffers (pinned), copies in the region
    e2e = None
    if cfg != "4" and args.e2e_steps > 0:
        w = c["elem_bytes"]
        src_h = values_torch(n, 99, w, "cpu").pin_memory()
        dst_h = torch.empty_like(src_h).pin_memory()
        # host API converts whole layout instances; use the per-tile layout + batch for chunking
        from workloads import configs as _cf
        if cfg == "2":
            ct = _cf.cfg2(batch_bits=0)
            At, Bt = ll.Layout.from_spec(ct["A"]), ll.Layout.from_spec(ct["B"])
            nb = n >> 14
        else:
            At, Bt, nb = A, B, 1
        # scratch: 2 slots x 16 MiB per side (the library chunks by instances or shards);
        # layouts that cannot be chunked need the whole buffer
        try:
            ll.shard_describe(At, Bt, 8 * w, 2, 0)
            shardable = True
        except ll.LLError:
            shardable = False
        scratch = min(n * w, 32 << 20) if (nb > 1 or shardable) else n * w
        ds = torch.empty(scratch, dtype=torch.uint8, device=dev)
        dd = torch.empty(scratch, dtype=torch.uint8, device=dev)
        ll.convert_host(src_h, At, dst_h, Bt, 8 * w, nb, ds, dd, scratch)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            ll.convert_host(src_h, At, dst_h, Bt, 8 * w, nb, ds, dd, scratch, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * nbytes / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": n * w, "d2h_bytes_per_step": n * w,
               "ms_per_step": e_ms, "api": "ll_convert_host (pinned host buffers, 16 MiB chunks, copy-in/compute/copy-out streams)"}

    if cfg == "4" and args.e2e_steps > 0:
        # the gather end to end: values and indices in, results out (host
        # buffers, pinned), chunked by [128, 32] instances of the same layout
        from workloads import configs as _cf
        ct = _cf.cfg4(r_bits=0)
        Lt = ll.Layout.from_spec(ct["L"])
        nb = n >> Lt.in_bits
        src_h = values_torch(n, 98, 4, "cpu").pin_memory()
        idx_h = indices_torch(n, 97, 32, "cpu").pin_memory()
        out_h = torch.empty_like(src_h).pin_memory()
        scratch = 32 << 20
        dbuf = [torch.empty(scratch, dtype=torch.uint8, device=dev) for _ in range(3)]
        ll.gather_host(src_h, idx_h, out_h, Lt, ct["axis"], 32, nb, *dbuf, scratch)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            ll.gather_host(src_h, idx_h, out_h, Lt, ct["axis"], 32, nb, *dbuf, scratch, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * nbytes / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 4 * n,
               "ms_per_step": e_ms, "api": "ll_gather_host (pinned host buffers, 16 MiB chunks, copy-in/compute/copy-out streams)"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(cfg, c)
            except Exception as ex:  # the baseline must never break the line
                cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "oracle",
                       "sample": "failed: %s" % ex}
        generic_smem = "smem_jit=0" in args.tune
        if args.upcast:
            up_jit = "upcast_jit=0" not in args.tune
            smem_kernel = "ll_upcast_hbm (NVRTC)" if up_jit else "convert_smem_kernel (upcast)"
        else:
            smem_kernel = "convert_smem_kernel" if generic_smem else "ll_smem_hbm (NVRTC)"
        kernel = {"smem": smem_kernel,
                  "generic": "convert_generic_kernel",
                  "shuffle": "gather_shuffle_kernel" if cfg == "4" else "ll_shfl_hbm (NVRTC)",
                  "smem_noswizzle": "convert_smem_kernel", "smem_padded": "convert_smem_kernel",
                  "smem_async": "convert_async_kernel", "smem_tma": "convert_tma_kernel",
                  "regs": "convert_regs_kernel", "smem_tma_store": "convert_tma_store_kernel",
                  "copy": "cudaMemcpyAsync",
                  "direct": "gather_direct_kernel"}.get(plan.get("path"), plan.get("path"))
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "fp16" if cfg in ("1", "2") else
            {"3": "bf16", "4": "fp32", "5": "u8"}[cfg], "data": "synthetic",
            "config": {"workload": desc, "bytes_per_step_per_gpu": nbytes,
                       "l2": "%d rotating buffer sets, footprint %.0f MiB > 126 MB L2" % (
                           len(sets), sum(t.numel() * t.element_size() for s in sets for t in s) / 2**20),
                       "path": plan.get("path"), "granule_bytes": plan.get("granule_bytes"),
                       "tile_bits": len(plan.get("tile_dst_bits") or []) or None,
                       "pred_wavefronts_per_sts": plan.get("pred_wavefronts_per_sts"),
                       "pred_wavefronts_per_lds": plan.get("pred_wavefronts_per_lds"),
                       "tma": plan.get("tma"), "tune": args.tune or None,
                       "parallelism": "dp%d" % world},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic(cfg + ("_upcast" if args.upcast else "") +
                                                {"smem": ("_jit" if "upcast_jit=0" not in args.tune else "") if args.upcast
                                                 else ("" if "smem_jit=0" in args.tune else "_jit"), "smem_tma": "_tma", "regs": "_regs", "smem_tma_store": "_tmas",
                                                 "shuffle": "_shfl"}.get(
                                                    plan.get("path"), "")),
                         "peak_source": peak_src, "kernel": kernel,
                         "avg_launch_us": avg_launch_ms * 1000,
                         "frac_of_8TBs": achieved / 8000.0},
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "timing": "CUDA graph of K steps replayed once" if graph is not None else "K launches from Python",
            "e2e": e2e,
            "cpu_baseline": cpu,
            "verify": verify,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
