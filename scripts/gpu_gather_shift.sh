#!/bin/bash
O=gpurun_out/gather_shift; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather or generic" > $O/pytest.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --config 4"
for r in 1 2; do
  timeout 300 python bench.py $B > $O/direct_r$r.json 2>/dev/null
  timeout 300 python bench.py $B --path shuffle > $O/shfl_r$r.json 2>/dev/null
  for v in 2 8; do timeout 300 python bench.py $B --path shuffle --tune gather_vpt=$v > $O/shfl_v${v}_r$r.json 2>/dev/null; done
  timeout 300 python bench.py $B --tune gather_v8=1 > $O/direct_v8_r$r.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config 2 --path generic > $O/cfg2_generic_r$r.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['value']),d['clocks']['sm_mhz'])"; done > $O/summary.txt
tail -2 $O/pytest.txt >> $O/summary.txt
