#!/bin/bash
# ll_convert_host with pitched shards (transpose e2e) vs the whole-instance path.
O=gpurun_out/host2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "convert_host or shard" > $O/pytest.txt 2>&1
for r in 1 2; do for h in 1 0; do
  timeout 300 python bench.py --config 3 --no-cpu-baseline --e2e-steps 10 --tune host_2d=$h > $O/cfg3_h${h}_r$r.json 2>$O/cfg3_h${h}_r$r.err
done; done
timeout 300 python bench.py --config 2 --no-cpu-baseline --e2e-steps 10 > $O/cfg2.json 2>/dev/null
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['value']),d['e2e'])"; done > $O/summary.txt
tail -2 $O/pytest.txt >> $O/summary.txt
