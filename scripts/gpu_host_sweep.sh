#!/bin/bash
# ll_convert_host chunk size x slots (e2e GB/s), configs 2 and 3.
O=gpurun_out/host_sweep; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for c in 2 3; do for mb in 4 8 16 32; do for sl in 2 3 4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 10 \
    --tune host_chunk_mb=$mb --tune host_slots=$sl > $O/cfg${c}_mb${mb}_s$sl.json 2>/dev/null
done; done; done
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['e2e']['value'],1))"; done > $O/summary.txt
