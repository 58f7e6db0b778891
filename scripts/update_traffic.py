"""Merge one run's ncu_summary.json (scripts/ncu_summary.py output) into
profiles/ncu_traffic.json, the per-kernel DRAM bytes bench.py reports as
roofline.traffic.  Keys: prof_<key>.ncu-rep -> "<key>".

usage: python scripts/update_traffic.py profiles/r01/final9/ncu_summary.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path):
    run = os.path.basename(os.path.dirname(path))
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(dst)) if os.path.exists(dst) else {}
    for r in json.load(open(path)):
        key = os.path.basename(r["report"])[len("prof_"):-len(".ncu-rep")]
        rd, wr = r.get("dram_read_MB"), r.get("dram_write_MB")
        if rd is None or wr is None:
            continue
        d[key] = {
            "kernel": r["kernel"],
            "dram_bytes_per_launch": int(round((rd + wr) * 1e6)),
            "dram_read_bytes": int(round(rd * 1e6)),
            "dram_write_bytes": int(round(wr * 1e6)),
            "note": "one ncu --set full capture (cold, replayed; profiles/r01/%s); writes still "
                    "dirty in L2 at kernel end are not counted" % run,
            "smem_ld_wavefronts_per_inst": r.get("smem_ld_wavefronts_per_inst"),
            "smem_st_wavefronts_per_inst": r.get("smem_st_wavefronts_per_inst"),
        }
    json.dump(d, open(dst, "w"), indent=1)
    print("updated", sorted(d))


if __name__ == "__main__":
    main(sys.argv[1])
