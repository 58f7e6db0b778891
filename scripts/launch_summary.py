"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
launches, total and average microseconds per kernel name, and the share of
the repository's own kernels (ll_* / convert_* / gather_* / checksum_*).

    python scripts/launch_summary.py launches.csv "what was run" > summary.json
"""
import csv
import json
import sys

OWN = ("ll_", "convert_", "gather_", "checksum_", "void ll::")


def main():
    path, what = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    k = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"][:60]
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1000.0 if r["Metric Unit"] in ("nsecond", "ns") else (v * 1000.0 if r["Metric Unit"] in ("msecond", "ms") else v)
        e = k.setdefault(name, {"launches": 0, "total_us": 0.0})
        e["launches"] += 1
        e["total_us"] += us
    own = {n: e for n, e in k.items() if n.startswith(OWN) or "ll_" in n.split("(")[0]}
    for e in k.values():
        e["total_us"] = round(e["total_us"], 1)
        e["avg_us"] = round(e["total_us"] / e["launches"], 2)
    tot = sum(e["total_us"] for e in k.values())
    print(json.dumps({"what": what, "kernels": k, "own_kernels": sorted(own),
                      "own_share_of_time": round(sum(e["total_us"] for e in own.values()) / tot, 4) if tot else None},
                     indent=1))


if __name__ == "__main__":
    main()
