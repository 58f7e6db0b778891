"""Benchmark of the hot path: layout conversion (and gather) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Default workload = the largest single-GPU config of BASELINE.json,
configs[4] ("cfg5"): the mxfp4 packed [32768, 16384] u8 tensor converted from
the coalesced blocked byte layout to the packed mma A-fragment image (reading
A22), 512 MiB in + 512 MiB out per step.  The same run also times configs 2,
3 and 4 ("also", fewer steps) so every config has a driver-measured line.

One step = one ll_convert over the whole tensor (planning is cached on the
host; the kernel does the rest).  Inputs are synthetic (seeded splitmix64
patterns generated on the device).  Timing: W untimed warm-up steps, then K
steps bracketed by a barrier and torch.cuda.synchronize(); the K steps are
captured as R (<= 10) CUDA graphs of consecutive steps, replayed back to back
with CUDA events between them on the launching stream, so the line carries
the whole-region value and the median / spread of the R replays (P:739:
median of 10).  Buffer sets rotate so the footprint exceeds the 126 MB L2.

Multi-GPU: one process per GPU.  `--gpus N` without WORLD_SIZE in the
environment launches N ranks itself (torch.distributed.run, 127.0.0.1);
under torchrun WORLD_SIZE must equal N.  N > 1 defaults to strong scaling of
cfg5: rank r converts shard r of the top block bits (ll_convert_shard, its
own slices of src and dst, no collective on the data path); time = max over
ranks of the device-timed region.  `--dist-backend gloo` runs the same flow
with several ranks on one GPU (tests of the multi-rank plumbing).

Measured shared-memory wavefronts and DRAM bytes of the dominant kernels
come from an ncu subprocess of this very run (`--ncu auto`, N = 1, rank 0):
`bench.py --ncu-probe` executes one launch per config under
`ncu --metrics ...` and the line reports its counters.

Prints ONE JSON line (rank 0).
"""

import argparse
import csv
import io
import json
import os
import shutil
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "convert_layout effective GB/s vs 8 TB/s HBM peak; smem bank conflicts/request"
CONFIGS = ["1", "2", "3", "4", "4full", "5", "6"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="5", choices=CONFIGS)
    ap.add_argument("--path", default="auto")
    ap.add_argument("--upcast", action="store_true",
                    help="config 5 only: fused mxfp4 dequantisation to bf16 (NEXT #1)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="strong (default for cfg2/cfg5): rank r converts shard r of the top "
                         "block bits (ll_convert_shard); weak: every rank converts the whole "
                         "workload")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-gather-scratch-mb", type=int, default=32,
                    help="device staging per buffer for ll_gather_host")
    ap.add_argument("--e2e-scratch-mb", type=int, default=64,
                    help="device staging per side for ll_convert_host (2 slots of its 32 MiB chunks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--also", default="2,3,4",
                    help="extra configs timed in the same run (N = 1; '' = none)")
    ap.add_argument("--also-steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=10, help="graph replays the K steps are split into")
    ap.add_argument("--ncu", default="auto", choices=["auto", "on", "off"],
                    help="measure smem wavefronts / DRAM bytes in an ncu subprocess (N = 1)")
    ap.add_argument("--ncu-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe-configs", default="", help=argparse.SUPPRESS)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--tune", action="append", default=[], metavar="KNOB=VALUE",
                    help="ll_tune knob before planning (e.g. tma_stages=4); repeatable")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch each step from Python instead of replaying CUDA graphs")
    return ap.parse_args(argv)


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
    elif cfg == "4full":
        c = configs.cfg4(variant="full")
        desc = "cfg4 full-axis variant: tl.gather along the 4096-long axis of [4096,4096] fp32, int32 idx in [0,4096)"
    elif cfg == "6":
        c = configs.cfg6()
        desc = ("cfg6: HBM pre-shuffle of a bf16 [8192,8192] operand, row-major -> mma m16n8k16 "
                "B-fragment order, 16 B per thread (P:558-563, reading A25)")
    else:
        c = configs.cfg5()
        desc = "cfg5: mxfp4 packed [32768,16384] u8, blocked -> packed mma A-fragment (reading A22)"
    return c, desc


def is_gather(cfg):
    return cfg.startswith("4")


def algorithmic_bytes(cfg, c):
    """w read + w written per element; gather + 4 B of index."""
    from workloads.configs import total_elems
    if is_gather(cfg):
        n = total_elems(c["L"])
        return n * c["elem_bytes"] * 2 + n * 4
    return total_elems(c["A"]) * c["elem_bytes"] + total_elems(c["B"]) * c["elem_bytes"]


DTYPE = {"1": "fp16", "2": "fp16", "3": "bf16", "4": "fp32", "4full": "fp32", "5": "u8", "6": "bf16"}


# ------------------------------------------------------------------- clocks

class ClockSampler:
    """NVML polling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index=0, period=0.0005):
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

    def _sample(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
        }
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

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join()
            self._sample()

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
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy_ of 2 GiB)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def git_head():
    try:
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                              capture_output=True, text=True, timeout=10).stdout.strip() or None
    except Exception:
        return None


def split_reps(K, R):
    """K steps into R consecutive groups (sizes differ by at most one)."""
    R = max(1, min(R, K))
    base, extra = divmod(K, R)
    out, s = [], 0
    for i in range(R):
        n = base + (1 if i < extra else 0)
        out.append((s, s + n))
        s += n
    return out


# --------------------------------------------------------------- CPU baseline

def _cfg5_shard_worker(args):
    """One process of the cfg5 CPU baseline: converts its shard (rows of the
    top block bits) with the oracle until the budget is spent; returns
    (reps, seconds, bytes per rep, indexed checksum of the shard's dst)."""
    shard, n_shards, m_bits, kb_bits, budget = args
    from oracle import checksum as ock
    from oracle import convert as oconv
    from oracle.layout import Layout as OL
    from workloads import configs
    from workloads.values import values_np
    sb = n_shards.bit_length() - 1
    cs = configs.cfg5(m_bits=m_bits - sb, kb_bits=kb_bits)      # one shard = fewer top m bits
    A, B = OL(**cs["A"]), OL(**cs["B"])
    n = 1 << A.in_bits
    src = values_np(n, 7, 1, start=shard * n)
    reps, t0 = 0, time.time()
    while True:
        dst = oconv.convert_np(src, A, B)
        reps += 1
        if time.time() - t0 > budget:
            break
    dt = time.time() - t0
    ck = ock.checksum_np(dst, indexed=True, base=shard * n)
    return reps, dt, 2 * n, "%016x" % ck


def cpu_baseline(cfg, c, budget_s=12.0):
    """The oracle as it stands (oracle.convert.convert_np / gather_np, the
    plain definition) on a bounded sample of the workload, scaled to the
    metric's unit: cfg1 in ms per conversion; cfg2-4
    one process; cfg5 a process pool of os.cpu_count() workers, one shard of
    the sample each, with per-shard checksums."""
    import numpy as np
    from oracle import convert as oconv
    from oracle.layout import Layout as OL
    from workloads import configs
    from workloads.values import indices_np, values_np
    cores = os.cpu_count() or 1
    if cfg == "5":
        import multiprocessing as mp
        m_bits, kb_bits = 12, 10           # sample: 4 MiB of the packed tensor
        n_sh = 1 << (max(1, cores).bit_length() - 1)
        n_sh = max(1, min(n_sh, 1 << (m_bits - 7)))
        t0 = time.time()
        with mp.get_context("spawn").Pool(n_sh) as pool:
            res = pool.map(_cfg5_shard_worker,
                           [(s, n_sh, m_bits, kb_bits, budget_s) for s in range(n_sh)])
        wall = time.time() - t0
        tot = sum(r[0] * r[2] for r in res)
        slowest = max(r[1] for r in res)
        return {"value": tot / slowest / 1e9, "unit": "GB/s", "cores": n_sh, "kind": "oracle",
                "sample": "cfg5 layouts with m_bits=%d kb_bits=%d (%d elements), %d shards of "
                          "the top block bits, convert_np repeated per worker for %.0f s"
                          % (m_bits, kb_bits, 1 << (m_bits + kb_bits), n_sh, budget_s),
                "host_cpus": cores, "seconds": round(wall, 2),
                "per_shard": [{"reps": r[0], "s": round(r[1], 2), "checksum": r[3]} for r in res],
                "single_core_s_per_shard": round(sum(r[1] / r[0] for r in res) / len(res), 4)}
    t0 = time.time()
    if cfg == "1":
        cs = configs.cfg1("mma")
        A, B = OL(**cs["A"]), OL(**cs["B"])
        src = values_np(1 << A.in_bits, 7, 2)
        reps, t0 = 0, time.time()
        while time.time() - t0 < min(budget_s, 5.0):
            oconv.convert_np(src, A, B)
            reps += 1
        dt = time.time() - t0
        return {"value": dt / reps * 1e3, "unit": "ms", "cores": 1, "kind": "oracle",
                "sample": "%d x convert_np on the whole cfg1 tensor (256 elements)" % reps,
                "host_cpus": cores, "seconds": round(dt, 2),
                "gbps": reps * 1024 / dt / 1e9}
    if is_gather(cfg):
        full = cfg == "4full"
        cs = configs.cfg4(r_bits=1, variant="full") if full else configs.cfg4(r_bits=6)
        L = OL(**cs["L"])
        n = 1 << L.in_bits
        src = values_np(n, 4, 4)
        idx = indices_np(n, 5, cs["idx_limit"])
        reps, t0 = 0, time.time()
        while True:
            oconv.gather_np(src, idx, L, cs["axis"])
            reps += 1
            if time.time() - t0 > budget_s:
                break
        dt = time.time() - t0
        return {"value": reps * n * 12 / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
                "sample": "%d x gather_np on %s (%d elements)" % (reps, cs["name"], n),
                "host_cpus": cores, "seconds": round(dt, 2)}
    if cfg == "2":
        cs = configs.cfg2(batch_bits=4)
    elif cfg == "6":
        cs = configs.cfg6(n_bits=10, k_bits=10)
    else:
        cs = configs.cfg3(n_bits=10)
    A, B = OL(**cs["A"]), OL(**cs["B"])
    n = 1 << A.in_bits
    w = cs["elem_bytes"]
    src = values_np(n, 7, w)
    reps, t0 = 0, time.time()
    while True:
        oconv.convert_np(src, A, B)
        reps += 1
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    return {"value": reps * n * w * 2 / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": "%d x convert_np on %s (%d elements)" % (reps, cs.get("name"), n),
            "host_cpus": cores, "seconds": round(dt, 2)}


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The tier's reference arm: the oracle timed on the host cores (rank 0
    only; other ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = args.config
    c, desc = workload(cfg)
    budget = max(1.0, min(20.0, 90.0 / max(1, args.steps)))
    vals = [cpu_baseline(cfg, c, budget_s=budget) for _ in range(max(1, args.steps))]
    v = sum(x["value"] for x in vals) / len(vals)
    b0 = vals[0]
    unit = b0["unit"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(x["seconds"] for x in vals) * 1000 / len(vals),
            "higher_is_better": unit != "ms", "scaling": "strong" if cfg in ("2", "5") else "weak",
            "vs_baseline": None, "dtype": DTYPE[cfg], "data": "synthetic",
            "config": {"workload": desc, "sample": b0["sample"]},
            "cpu_baseline": {"value": v, "unit": unit, "cores": b0["cores"], "kind": "oracle",
                             "sample": b0["sample"], "host_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ncu probe

NCU_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
]
OUR_KERNELS = "regex:(ll_smem|ll_shfl|ll_upcast|ll_regs|ll_regperm|ll_tma|ll_gather|convert_.*kernel|gather_.*kernel)"


def ncu_probe(args):
    """Child of the ncu subprocess: one launch per config (AUTO plan), nothing
    else of ours."""
    import torch
    import paper_2505_23819_b200 as ll
    from workloads.values import indices_torch, values_torch
    for kv in args.tune:
        k, v = kv.split("=")
        ll.tune(k, int(v))
    dev = torch.device("cuda", 0)
    for cfg in args.probe_configs.split(","):
        c, _ = workload(cfg)
        if is_gather(cfg):
            L = ll.Layout.from_spec(c["L"])
            n = 1 << L.in_bits
            s = values_torch(n, 4, 4, dev)
            i = indices_torch(n, 5, c["idx_limit"], dev)
            ll.gather(s, i, torch.empty_like(s), L, c["axis"], 32, path=args.path)
        else:
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            w = c["elem_bytes"]
            s = values_torch(1 << A.in_bits, 7, w, dev)
            d = torch.empty(1 << B.in_bits, dtype=s.dtype, device=dev)
            if args.upcast and cfg == "5":
                sc = (indices_torch(s.numel() // 16, 42, 16, dev) + 120).to(torch.uint8)
                d = torch.empty(2 * s.numel(), dtype=torch.int16, device=dev)
                ll.mxfp4_upcast(s, A, sc, d, B)
            else:
                ll.convert(s, A, d, B, 8 * w, path=args.path)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


def run_ncu(args, cfgs, timeout=240):
    """ncu --metrics over one launch per config in a subprocess; returns
    {cfg: {metric: value}} or {"error": ...}."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    cmd = [ncu, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none",
           "--kernel-name", OUR_KERNELS, "--csv", "--page", "raw",
           sys.executable, os.path.abspath(__file__), "--ncu-probe",
           "--probe-configs", ",".join(cfgs), "--path", args.path]
    if args.upcast:
        cmd.append("--upcast")
    for kv in args.tune:
        cmd += ["--tune", kv]
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except Exception as ex:
        return {"error": "ncu subprocess: %s" % ex}
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith('"')]
    if p.returncode != 0 or len(lines) < 3:
        return {"error": "ncu rc=%d: %s" % (p.returncode, (p.stderr or p.stdout)[-300:])}
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    if len(vals) != len(cfgs):
        return {"error": "ncu: %d kernels profiled for %d configs" % (len(vals), len(cfgs))}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
             "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    out = {}
    for cfg, row in zip(cfgs, vals):
        d = {"kernel": row[hdr.index("Kernel Name")][:60]}
        for m in NCU_METRICS:
            if m in hdr:
                j = hdr.index(m)
                try:
                    x = float(row[j].replace(",", ""))
                except ValueError:
                    continue
                d[m] = x * scale.get(units[j], 1)
        out[cfg] = d
    return out


def smem_summary(ncu_row, plan):
    """Measured wavefronts per shared-memory request (ncu) vs the planner's
    optimum (the lemma's n per request)."""
    if not ncu_row or "error" in ncu_row:
        return None
    g = ncu_row.get
    sts, lds = g("smsp__sass_inst_executed_op_shared_st.sum"), g("smsp__sass_inst_executed_op_shared_ld.sum")
    if not sts and not lds:
        return {"kernel": ncu_row.get("kernel"), "sts": 0, "lds": 0,
                "note": "no shared-memory instructions in the dominant kernel"}
    res = {"kernel": ncu_row.get("kernel"), "sts": sts, "lds": lds,
           "wavefronts_per_sts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum") / sts if sts else None,
           "wavefronts_per_lds": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum") / lds if lds else None,
           "bank_conflicts_st": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
           "bank_conflicts_ld": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
           "optimum_per_sts": plan.get("pred_wavefronts_per_sts"),
           "optimum_per_lds": plan.get("pred_wavefronts_per_lds")}
    if res["optimum_per_sts"] and res["wavefronts_per_sts"]:
        res["excess_sts"] = res["wavefronts_per_sts"] / res["optimum_per_sts"]
    if res["optimum_per_lds"] and res["wavefronts_per_lds"]:
        res["excess_lds"] = res["wavefronts_per_lds"] / res["optimum_per_lds"]
    return res


# ----------------------------------------------------------------- self-launch

def self_launch(args):
    """`--gpus N` with no WORLD_SIZE: run N ranks of this script through
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------- our arm

class Bench:
    """One config's buffers, step function and plan, on this rank."""

    def __init__(self, ll, cfg, args, dev, world, rank, scaling, upcast=False):
        import torch
        from workloads.values import indices_torch, values_torch
        self.cfg, self.c, self.desc = cfg, *workload(cfg)
        c = self.c
        self.nbytes = algorithmic_bytes(cfg, c)
        self.sharded = scaling == "strong" and world > 1
        self.upcast = upcast
        path = args.path
        if is_gather(cfg):
            L = ll.Layout.from_spec(c["L"])
            n = 1 << L.in_bits
            self.n = n
            self.sets = [(values_torch(n, 4 + s + 10 * rank, 4, dev),
                          indices_torch(n, 5 + s, c["idx_limit"], dev),
                          torch.empty(n, dtype=torch.int32, device=dev)) for s in range(2)]
            self.L = L

            def step(i):
                s, ix, o = self.sets[i % 2]
                ll.gather(s, ix, o, L, c["axis"], 32, path=path)
            self.plan = ll.gather_describe(L, c["axis"], 32, path)
            self.dst_index = 2
        else:
            A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
            self.A, self.B = A, B
            w = c["elem_bytes"]
            n = 1 << A.in_bits
            self.n = n
            if self.sharded:
                s0, s1, d0, d1 = ll.shard_describe(A, B, 8 * w, world, rank, path)
                n_loc = (s1 - s0) // w
                self.nbytes = (s1 - s0) + (d1 - d0)
                self.shard = (s0, s1, d0, d1)
            else:
                n_loc = n
            self.n_loc = n_loc
            per_set = 2 * n_loc * w * (3 if upcast else 1)
            nsets = 2 if per_set >= (256 << 20) else min(64, -(-(512 << 20) // per_set) + 1)
            dt = values_torch(1, 0, w, "cpu").dtype
            self.sets = [(values_torch(n_loc, 7 + s + 10 * rank, w, dev, start=rank * n_loc),
                          torch.empty(n_loc, dtype=dt, device=dev)) for s in range(nsets)]
            if upcast:
                n_sc = n // 16
                self.scales = (indices_torch(n_sc, 42, 16, dev) + 120).to(torch.uint8)
                self.sets = [(s_, torch.empty(2 * n_loc, dtype=torch.int16, device=dev))
                             for s_, _ in self.sets]
                # 1 B packed read + 1/16 B scale + 4 B of bf16 written per packed byte
                self.nbytes = n * w + n_sc + 4 * n * w

            def step(i):
                s, d = self.sets[i % len(self.sets)]
                if upcast:
                    ll.mxfp4_upcast(s, A, self.scales, d, B)
                elif self.sharded:
                    ll.convert_shard(s, A, d, B, 8 * w, world, rank, path=path)
                else:
                    ll.convert(s, A, d, B, 8 * w, path=path)
            self.plan = ll.plan_describe(A, B, 8 * w, path)
            self.dst_index = 1
        self.step = step

    def footprint_mib(self):
        return sum(t.numel() * t.element_size() for s in self.sets for t in s) / 2**20


def time_steps(ll, b, K, warmup, R, use_graph, world, sync_barrier, clk=None):
    """W warm-up steps, then exactly K steps split into R consecutive groups,
    each a CUDA graph (or plain launches) between CUDA events on the launching
    stream.  Returns (total_ms, per-group ms list, per-group step counts,
    launches counted in the timed region)."""
    import torch
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    for i in range(max(3, warmup)):
        b.step(i)
    torch.cuda.synchronize()
    groups = split_reps(K, R)
    graphs = []
    l0 = ll.launch_count()
    if use_graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        for g0, g1 in groups:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    for i in range(g0, g1):
                        b.step(i)
            graphs.append(g)
        stream.wait_stream(cap)
        launches = ll.launch_count() - l0
        graphs[0].replay()                       # warm the graph machinery
        torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(groups) + 1)]
    sync_barrier()
    torch.cuda.synchronize()
    import contextlib
    with (clk if clk is not None else contextlib.nullcontext()):
        ev[0].record(stream)
        for gi, (g0, g1) in enumerate(groups):
            if use_graph:
                graphs[gi].replay()
            else:
                for i in range(g0, g1):
                    b.step(i)
            ev[gi + 1].record(stream)
        torch.cuda.synchronize()
    sync_barrier()
    if not use_graph:
        launches = ll.launch_count() - l0
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(groups))]
    total = ev[0].elapsed_time(ev[-1])
    return total, per, [g1 - g0 for g0, g1 in groups], launches


def median(xs):
    s = sorted(xs)
    n = len(s)
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


def main():
    args = parse()
    if args.ncu_probe:
        ncu_probe(args)
        return
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(self_launch(args))
    world = int(env_world or "1")
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d: under torchrun --gpus must "
                         "equal --nproc-per-node (or run without torchrun to self-launch)"
                         % (args.gpus, world))
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_2505_23819_b200 as ll
    from paper_2505_23819_b200 import multigpu
    for kv in args.tune:
        k, v = kv.split("=")
        ll.tune(k, int(v))

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device")
    if world > ndev and args.dist_backend == "nccl":
        raise SystemExit("bench.py: %d ranks but %d visible GPUs (use --dist-backend gloo to "
                         "share one GPU in a plumbing test)" % (world, ndev))
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    gloo = args.dist_backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    coll_dev = None if gloo else dev

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = args.config
    if args.upcast and (cfg != "5" or world > 1):
        raise SystemExit("--upcast is config 5 on one GPU only")
    scaling = args.scaling or ("strong" if cfg in ("2", "5") else "weak")
    if scaling == "strong" and is_gather(cfg) and world > 1:
        raise SystemExit("strong scaling is implemented for the conversions (cfg2 / cfg5)")
    b = Bench(ll, cfg, args, dev, world, rank, scaling, upcast=args.upcast)
    stream = torch.cuda.current_stream()
    K = args.steps
    clk = ClockSampler(local_dev)
    total_ms, per_ms, per_n, launches = time_steps(ll, b, K, args.warmup, args.reps,
                                                   not args.no_graph, world, barrier, clk)
    total_ms = multigpu.max_over_ranks(total_ms, device=coll_dev)
    ms_per_step = total_ms / K
    bytes_all = multigpu.gather_records([b.nbytes], device=coll_dev)
    value = multigpu.aggregate_gbps([r[0] for r in bytes_all], [ms_per_step] * world, scaling)
    rep_gbps = [b.nbytes * n / (t * 1e-3) / 1e9 for t, n in zip(per_ms, per_n)]
    achieved = b.nbytes / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # row a12 (untimed): checksum record of the last step's destination per
    # rank (ll_checksum, indexed), and for conversions the permutation
    # property on the whole buffer (index-free checksums of src and dst agree)
    last = b.sets[(K - 1) % len(b.sets)]
    dst_t = last[b.dst_index]
    ck = torch.zeros(3, dtype=torch.int64, device=dev)
    base = b.shard[2] // b.c["elem_bytes"] if b.sharded and not args.upcast else 0
    ll.checksum(dst_t, dst_t.numel(), 8 * dst_t.element_size(), ck[0:1], index_base=base,
                stream=stream)
    perm_check = not is_gather(cfg) and not args.upcast
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
              "how": "ll_checksum (row a12): indexed splitmix64 sum of the last step's destination "
                     "(shard checksums carry their slice's base, so they add up to the whole "
                     "buffer's); permutation_ok = index-free sums of src and dst agree; NCCL/gloo "
                     "all_gather_object after the timed region"}

    e2e = run_e2e(ll, b, args, dev, world, rank, scaling, barrier, coll_dev)

    # the other configs, same protocol, N = 1 only
    also = {}
    if world == 1 and args.also and not args.upcast:
        for ac in [x for x in args.also.split(",") if x and x != cfg]:
            try:
                ab = Bench(ll, ac, args, dev, 1, 0, "weak")
                t, pm, pn, _ = time_steps(ll, ab, args.also_steps, 5, args.reps, not args.no_graph,
                                          1, barrier)
                msps = t / args.also_steps
                v = ab.nbytes / (msps * 1e-3) / 1e9
                rg = [ab.nbytes * n / (x * 1e-3) / 1e9 for x, n in zip(pm, pn)]
                also["cfg" + ac] = {"workload": ab.desc, "value": v, "unit": "GB/s",
                                    "ms_per_step": msps, "steps": args.also_steps,
                                    "frac": v / peak, "frac_of_8TBs": v / 8000.0,
                                    "median_gbps": median(rg), "min_gbps": min(rg),
                                    "max_gbps": max(rg), "path": ab.plan.get("path"),
                                    "bytes_per_step": ab.nbytes, "_plan": ab.plan,
                                    "footprint_mib": round(ab.footprint_mib())}
                del ab
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
            except Exception as ex:
                also["cfg" + ac] = {"error": str(ex)[:200]}

    ncu = {}
    if rank == 0 and world == 1 and (args.ncu == "on" or (args.ncu == "auto" and not args.no_graph)):
        cfgs = [cfg] + [k[3:] for k in also if "error" not in also[k]]
        ncu = run_ncu(args, cfgs)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(cfg, b.c)
            except Exception as ex:  # the baseline must never break the line
                cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "oracle",
                       "sample": "failed: %s" % ex}
        main_ncu = ncu.get(cfg) if "error" not in ncu else None
        kern = (main_ncu or {}).get("kernel") or kernel_name(b.plan, cfg, args)
        traffic = None
        if main_ncu and "dram__bytes_read.sum" in main_ncu:
            traffic = main_ncu["dram__bytes_read.sum"] + main_ncu.get("dram__bytes_write.sum", 0)
        for k, a in also.items():
            if "error" in a:
                continue
            plan = a.pop("_plan")
            row = ncu.get(k[3:]) if "error" not in ncu else None
            a["smem"] = smem_summary(row, plan) if row else None
            if row and "dram__bytes_read.sum" in row:
                a["ncu_dram_bytes"] = row["dram__bytes_read.sum"] + row.get("dram__bytes_write.sum", 0)
                a["ncu_kernel_us_cold"] = row.get("gpu__time_duration.sum")
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None,
            "dtype": "bf16 out (u8 in)" if args.upcast else DTYPE[cfg], "data": "synthetic",
            "config": {"workload": b.desc + (" + fused mxfp4 -> bf16 upcast" if args.upcast else ""),
                       "bytes_per_step_per_gpu": b.nbytes,
                       "l2": "%d rotating buffer sets, footprint %.0f MiB > 126 MB L2 (no flush)" % (
                           len(b.sets), b.footprint_mib()),
                       "path": b.plan.get("path"), "granule_bytes": b.plan.get("granule_bytes"),
                       "tile_bits": len(b.plan.get("tile_dst_bits") or []) or None,
                       "tune": args.tune or None,
                       "parallelism": ("shard%d" if b.sharded else "dp%d") % world,
                       "dist_backend": args.dist_backend if world > 1 else None},
            "timing": {"how": ("K steps as %d CUDA graphs replayed back to back" % len(per_ms))
                       if not args.no_graph else "K launches from Python in %d groups" % len(per_ms),
                       "median_gbps": median(rep_gbps), "min_gbps": min(rep_gbps),
                       "max_gbps": max(rep_gbps), "reps": len(rep_gbps), "steps_per_rep": per_n[0],
                       "rank0_ms_per_rep": per_ms},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum, ncu "
                                           "subprocess of this run (writes under-counted: dirty L2 "
                                           "lines at kernel end)" if traffic else None,
                         "peak_source": peak_src, "kernel": kern,
                         "avg_launch_us": ms_per_step * 1000,
                         "frac_of_8TBs": achieved / 8000.0},
            "smem": smem_summary(main_ncu, b.plan) if main_ncu else
            ({"error": ncu.get("error")} if ncu else None),
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "verify": verify,
            "also": also or None,
            "head": git_head(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def kernel_name(plan, cfg, args):
    if args.upcast:
        return "ll_upcast_hbm (NVRTC)"
    tuned = dict(kv.split("=") for kv in args.tune)
    tma_jit = tuned.get("tma_jit", "1") != "0"
    if is_gather(cfg):
        return {"smem": "ll_gather_smem (NVRTC)", "shuffle": "ll_gather_shfl (NVRTC)",
                "generic": "gather_direct_kernel", "direct": "gather_direct_kernel"}.get(
                    plan.get("path"), plan.get("path"))
    return {"smem": "ll_smem_hbm (NVRTC)", "generic": "convert_generic_kernel",
            "shuffle": "ll_shfl_hbm (NVRTC)", "regperm": "ll_regperm (NVRTC)",
            "smem_tma": "ll_tma_hbm (NVRTC)" if tma_jit else "convert_tma_kernel",
            "regs": "convert_regs_kernel",
            "smem_tma_store": "ll_tma_hbm (NVRTC)" if tma_jit else "convert_tma_store_kernel",
            "copy": "cudaMemcpyAsync"}.get(plan.get("path"), plan.get("path"))


def run_e2e(ll, b, args, dev, world, rank, scaling, barrier, coll_dev):
    """The same metric end to end through the public API with HOST buffers
    (pinned): every step copies its inputs host -> device and its result
    device -> host inside the timed region."""
    import torch
    from workloads.values import indices_torch, values_torch
    if args.e2e_steps <= 0:
        return None
    cfg, c = b.cfg, b.c
    stream = torch.cuda.current_stream()
    E = args.e2e_steps

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(E):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return multigpu_max(e0.elapsed_time(e1) / E, coll_dev)

    if is_gather(cfg):
        # values and indices in, results out, chunked by whole instances
        from workloads import configs as _cf
        ct = _cf.cfg4(r_bits=0, variant="full" if cfg == "4full" else "tile")
        Lt = ll.Layout.from_spec(ct["L"])
        n = b.n
        nb = n >> Lt.in_bits
        src_h = values_torch(n, 98, 4, "cpu").pin_memory()
        idx_h = indices_torch(n, 97, ct["idx_limit"], "cpu").pin_memory()
        out_h = torch.empty_like(src_h).pin_memory()
        scratch = args.e2e_gather_scratch_mb << 20
        dbuf = [torch.empty(scratch, dtype=torch.uint8, device=dev) for _ in range(3)]
        ms = timed(lambda: ll.gather_host(src_h, idx_h, out_h, Lt, ct["axis"], 32, nb, *dbuf,
                                          scratch, stream=stream))
        return {"value": world * b.nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 4 * n, "ms_per_step": ms,
                "api": "ll_gather_host (pinned host buffers, %d MiB device staging per buffer, copy-in/"
                       "compute/copy-out streams)" % (scratch >> 20)}
    w = c["elem_bytes"]
    if b.upcast:
        # packed bytes + scales in, 2 GiB of bf16 out (copies, then the fused kernel)
        n = b.n
        pk_h = values_torch(n, 99, 1, "cpu").pin_memory()
        sc_h = b.scales.cpu().pin_memory()
        out_h = torch.empty(2 * n, dtype=torch.int16).pin_memory()
        pk_d, sc_d = torch.empty_like(b.sets[0][0]), torch.empty_like(b.scales)
        out_d = b.sets[0][1]

        def up():
            pk_d.copy_(pk_h, non_blocking=True)
            sc_d.copy_(sc_h, non_blocking=True)
            ll.mxfp4_upcast(pk_d, b.A, sc_d, out_d, b.B, stream=stream)
            out_h.copy_(out_d, non_blocking=True)
        ms = timed(up)
        return {"value": world * b.nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": n + n // 16, "d2h_bytes_per_step": 4 * n, "ms_per_step": ms,
                "api": "torch pinned copies + ll_mxfp4_upcast (sequential on one stream)"}
    if b.sharded:
        # this rank's shard: its slices in, its slice out
        s0, s1, d0, d1 = b.shard
        n_loc = b.n_loc
        src_h = values_torch(n_loc, 99, w, "cpu", start=rank * n_loc).pin_memory()
        dst_h = torch.empty(n_loc, dtype=src_h.dtype).pin_memory()
        scratch = min(s1 - s0, args.e2e_scratch_mb << 20)
        ds = torch.empty(scratch, dtype=torch.uint8, device=dev)
        dd = torch.empty(scratch, dtype=torch.uint8, device=dev)

        def sh():
            ll.convert_host_shard(src_h, b.A, dst_h, b.B, 8 * w, world, rank, ds, dd, scratch,
                                  stream=stream)
        ms = timed(sh)
        return {"value": world * b.nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": s1 - s0, "d2h_bytes_per_step": d1 - d0, "ms_per_step": ms,
                "api": "ll_convert_host_shard per rank (pinned host slices, %d MiB device staging per "
                       "side, copy-in/compute/copy-out streams)" % (scratch >> 20)}
    n = b.n
    src_h = values_torch(n, 99, w, "cpu").pin_memory()
    dst_h = torch.empty_like(src_h).pin_memory()
    from workloads import configs as _cf
    if cfg == "2":
        ct = _cf.cfg2(batch_bits=0)
        At, Bt = ll.Layout.from_spec(ct["A"]), ll.Layout.from_spec(ct["B"])
        nb = n >> 14
    else:
        At, Bt, nb = b.A, b.B, 1
    try:
        ll.shard_describe(At, Bt, 8 * w, 2, 0)
        shardable = True
    except ll.LLError:
        shardable = False
    scratch = min(n * w, args.e2e_scratch_mb << 20) if (nb > 1 or shardable) else n * w
    ds = torch.empty(scratch, dtype=torch.uint8, device=dev)
    dd = torch.empty(scratch, dtype=torch.uint8, device=dev)
    ms = timed(lambda: ll.convert_host(src_h, At, dst_h, Bt, 8 * w, nb, ds, dd, scratch,
                                       stream=stream))
    return {"value": world * b.nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": n * w, "d2h_bytes_per_step": n * w, "ms_per_step": ms,
            "api": "ll_convert_host (pinned host buffers, %d MiB device staging per side, 16-32 MiB "
                   "chunks, copy-in/compute/copy-out streams)" % (scratch >> 20)}


def multigpu_max(x, coll_dev):
    from paper_2505_23819_b200 import multigpu
    return multigpu.max_over_ranks(x, device=coll_dev)


if __name__ == "__main__":
    main()
