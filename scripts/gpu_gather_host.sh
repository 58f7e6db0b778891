#!/bin/bash
O=gpurun_out/gather_host; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host" > $O/pytest.txt 2>&1
for r in 1 2; do timeout 300 python bench.py --config 4 --no-cpu-baseline --e2e-steps 10 > $O/cfg4_r$r.json 2>$O/cfg4_r$r.err; done
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['value']),d['e2e'])"; done > $O/summary.txt
tail -2 $O/pytest.txt >> $O/summary.txt
