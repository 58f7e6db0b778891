#!/bin/bash
# PDL prefetch of the first K waves' tiles (knob pdl_prefetch_waves).
O=gpurun_out/r02s3p
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "hint_and_order" > $O/pytest.txt 2>&1
for c in 2 3 5; do
  timeout 900 python scripts/ab_knobs.py $c ";pdl_prefetch_waves=2;pdl_prefetch_waves=3" 5 >> $O/ab_waves.jsonl 2>> $O/ab.err
done
timeout 600 python scripts/shard_projection.py "" > $O/proj_default.jsonl 2>> $O/ab.err
timeout 600 python scripts/shard_projection.py "pdl_prefetch_waves=2" > $O/proj_w2.jsonl 2>> $O/ab.err
echo done > $O/done.txt
