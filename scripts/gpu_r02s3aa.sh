#!/bin/bash
# Smem conversion: prologue prefetch through the bulk-copy engine (knob pdl_prefetch_bulk).
O=gpurun_out/r02s3aa
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "hint_and_order" > $O/pytest.txt 2>&1
for c in 3 2 5; do
  timeout 900 python scripts/ab_knobs.py $c ";pdl_prefetch_bulk=1;pdl_prefetch=0" 5 >> $O/ab.jsonl 2>> $O/ab.err
done
timeout 600 python scripts/shard_projection.py "pdl_prefetch_bulk=1" > $O/proj_bulk.jsonl 2>> $O/ab.err
echo done > $O/done.txt
