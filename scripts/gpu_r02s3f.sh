#!/bin/bash
# PDL L2 prefetch, first wave only (pdl_prefetch=1) vs every CTA (=2):
# interleaved A/B on configs 3 / 2 / 5 / 6 and the shard projection.
O=gpurun_out/r02s3f
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "hint_and_order" > $O/pytest_knobs.txt 2>&1
for c in 3 2 5 6; do
  timeout 600 python scripts/ab_knobs.py $c ";pdl_prefetch=1;pdl_prefetch=2" 7 >> $O/ab_prefetch.jsonl 2>> $O/ab.err
done
timeout 600 python scripts/shard_projection.py "" > $O/proj_base.jsonl 2>> $O/ab.err
timeout 600 python scripts/shard_projection.py "pdl_prefetch=1" > $O/proj_prefetch1.jsonl 2>> $O/ab.err
timeout 600 python scripts/shard_projection.py "pdl_prefetch=2" > $O/proj_prefetch2.jsonl 2>> $O/ab.err
echo done > $O/done.txt
