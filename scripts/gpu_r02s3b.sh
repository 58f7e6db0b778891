#!/bin/bash
# Cache-hint ablation of the compiled smem kernel (knobs ld_hint / st_hint),
# interleaved A/B per config.
O=gpurun_out/r02s3b
mkdir -p $O
H=";ld_hint=1;ld_hint=2;ld_hint=3;st_hint=1;st_hint=2;st_hint=3;st_hint=4"
for c in 3 2 5; do
  timeout 600 python scripts/ab_knobs.py $c "$H" 5 >> $O/ab_hints.jsonl 2>> $O/ab_hints.err
done
echo done > $O/done.txt
