#!/bin/bash
# Check after the stall-capture / single-buffer / gather-unroll changes:
# smoke, the GPU suite, default bench lines, and the shuffle-gather A/B.
O=gpurun_out/final8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0"
for c in 2 3 4 5; do timeout 300 python bench.py --config $c $B > $O/bench_cfg$c.json 2>/dev/null; done
for rep in 1 2; do for u in 1 2; do for v in 2 4 8; do
  timeout 300 python bench.py --config 4 $B --path shuffle --tune gather_shfl_u=$u --tune gather_vpt=$v \
    > $O/g_u${u}_v${v}_r$rep.json 2>/dev/null
done; done; done
python - > $O/summary.txt <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/final8/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), round(d["value"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(os.path.basename(f), "ERR", str(e)[:80])
PY
tail -3 $O/pytest_gpu.txt >> $O/summary.txt; tail -2 $O/smoke.txt >> $O/summary.txt
