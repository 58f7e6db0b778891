#!/bin/bash
# Shuffle gather: warp-vectors in flight per thread (gather_shfl_u) x vectors per thread.
O=${O:-gpurun_out/gather_u}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k gather > $O/pytest.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do for u in 1 2 4; do for v in 2 4 8 16; do
  timeout 300 python bench.py --config 4 $B --path shuffle --tune gather_shfl_u=$u --tune gather_vpt=$v \
    > $O/g_u${u}_v${v}_r$rep.json 2>/dev/null
done; done; timeout 300 python bench.py --config 4 $B > $O/direct_r$rep.json 2>/dev/null; done
python - > $O/summary.txt <<'PY'
import json, glob, os
for f in sorted(glob.glob(os.environ.get("O", "gpurun_out/gather_u") + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(os.path.basename(f), round(d["value"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(os.path.basename(f), "ERR", str(e)[:80])
PY
tail -2 $O/pytest.txt >> $O/summary.txt
