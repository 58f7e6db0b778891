"""Print value / path / clock of bench JSON lines: python scripts/summ.py files..."""
import json
import sys

for f in sorted(sys.argv[1:]):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print("%-55s %9.1f  %-8s frac=%.3f  mhz=%s" % (f, d["value"], d["config"].get("path"),
              d["roofline"]["frac"], d["clocks"]["sm_mhz"]))
    except Exception as e:  # noqa: BLE001
        print("%-55s ERR %s" % (f, e))
