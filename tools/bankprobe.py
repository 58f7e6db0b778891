"""Drive tools/libbankprobe.so: one kernel launch per address pattern.

    python tools/bankprobe.py run  > manifest.json      (under ncu, see scripts/gpu_bankprobe.sh)
    python tools/bankprobe.py join manifest.json launches.csv

Patterns: synthetic checks of the phase model (reading A18) and the exact
per-lane shared-memory offsets of the planner's smem plans for configs 2, 3, 5.
"""
import ctypes
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def synthetic():
    P = []
    P.append(("w16_linear", 16, [[16 * l for l in range(32)]], 4))
    P.append(("w16_quarters_same_banks", 16, [[16 * (l % 8) + 1024 * (l // 8) for l in range(32)]], 4))
    P.append(("w16_2way_in_quarter", 16, [[16 * (l % 4) + 2048 * ((l // 4) % 2) + 4096 * (l // 8)
                                           for l in range(32)]], 8))
    P.append(("w16_8way_in_quarter", 16, [[128 * (l % 8) + 16 * (l // 8) for l in range(32)]], 32))
    P.append(("w8_linear", 8, [[8 * l for l in range(32)]], 2))
    P.append(("w8_halves_same_banks", 8, [[8 * (l % 16) + 1024 * (l // 16) for l in range(32)]], 2))
    P.append(("w4_linear", 4, [[4 * l for l in range(32)]], 1))
    P.append(("w4_stride128", 4, [[128 * l for l in range(32)]], 32))
    P.append(("w4_broadcast", 4, [[0 for l in range(32)]], 1))
    return P


def plan_patterns():
    import paper_2505_23819_b200 as ll
    from workloads import configs
    out = []
    for name, c in (("cfg2", configs.cfg2()), ("cfg3", configs.cfg3()), ("cfg5", configs.cfg5())):
        A, B = ll.Layout.from_spec(c["A"]), ll.Layout.from_spec(c["B"])
        d = ll.plan_describe(A, B, 8 * c["elem_bytes"])
        sb, g, G = d["smem_bytes"], d["group_warps_log2"], d["granule_bytes"]
        for side, thr, gran in (("sts", sb["sw_thr"], sb["sw_gran"]),
                                ("lds", sb["sr_thr"], sb["sr_gran"])):
            warps = []
            for w in range(1 << g):
                instrs = []
                for j in range(len(gran)):
                    row = []
                    for lane in range(32):
                        tb = lane | (w << 5)
                        x = 0
                        for b in range(5 + g):
                            if (tb >> b) & 1:
                                x ^= thr[b]
                        row.append(x ^ gran[j])
                    instrs.append(row)
                warps.append(instrs)
            ideal = max(1, G // 4)
            out.append(("%s_%s" % (name, side), G, warps, ideal, side == "sts"))
    return out


def run():
    import torch
    lib = ctypes.CDLL(os.path.join(HERE, "libbankprobe.so"))
    lib.bankprobe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    out = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    manifest = []

    def launch(name, width, store, warps_instrs, ideal, blocks=1):
        warps = len(warps_instrs)
        n_instr = len(warps_instrs[0])
        flat = [o for w in warps_instrs for ins in w for o in ins]
        t = torch.tensor(flat, dtype=torch.int64).to(torch.int32).cuda()
        st = lib.bankprobe(width, int(store), t.data_ptr(), warps, n_instr, 4, blocks,
                           out.data_ptr())
        manifest.append({"name": name, "width": width, "store": bool(store), "warps": warps,
                         "blocks": blocks, "n_instr": n_instr, "reps": 4,
                         "ideal_wavefronts_per_inst": ideal, "status": st})

    for name, width, pat, ideal in synthetic():
        launch(name, width, False, [[pat[0]]], ideal)
    for name, G, warps, ideal, store in plan_patterns():
        launch(name + "_1warp", G, store, warps[:1], ideal)
        launch(name + "_group", G, store, warps, ideal)
        launch(name + "_group_x8blocks", G, store, warps, ideal, blocks=8)
    print(json.dumps(manifest))


def join(manifest_path, csv_path):
    man = json.load(open(manifest_path))
    rows = [r for r in csv.DictReader(l for l in open(csv_path) if not l.startswith("=="))]
    per = {}
    for r in rows:
        if "probe" not in r["Kernel Name"]:
            continue
        per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = sorted(per)
    res = []
    for m, i in zip(man, ids):
        d = per[i]
        blocks, warps = m["blocks"], m["warps"]
        # the smem init loop issues 16384 / 32 = 512 warp-level 32-bit stores per block
        init_st = 512 * blocks
        if m["store"]:
            wf = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 0) - init_st
            ni = d.get("smsp__sass_inst_executed_op_shared_st.sum", 0) - init_st
        else:
            wf = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 0)
            ni = d.get("smsp__sass_inst_executed_op_shared_ld.sum", 0)
        m["measured_wavefronts_per_inst"] = (wf / ni) if ni else None
        m["raw"] = d
        res.append(m)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        res = join(sys.argv[2], sys.argv[3])
        for r in res:
            print("%-34s w=%2d %s warps=%d blocks=%d ideal=%d measured=%s" % (
                r["name"], r["width"], "st" if r["store"] else "ld", r["warps"], r["blocks"],
                r["ideal_wavefronts_per_inst"],
                "%.3f" % r["measured_wavefronts_per_inst"]
                if r["measured_wavefronts_per_inst"] is not None else None))
        if len(sys.argv) > 4:
            json.dump(res, open(sys.argv[4], "w"), indent=1)
