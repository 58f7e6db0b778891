#!/bin/bash
# bench.py vs ab_knobs on config 3 (methodology check), then the config-3
# tile-order sweep (knob tile_order: 10+k = k destination bits then the
# source order, 20+k = k source bits then the destination order).
O=gpurun_out/r02s3c
mkdir -p $O
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off"
for c in 3 2; do
  eval timeout 300 python bench.py --config $c $B --steps 300 > $O/bench_c${c}_300.json 2>/dev/null
  timeout 300 python scripts/ab_knobs.py $c "" 3 >> $O/ab_plain.jsonl 2>> $O/ab.err
  eval timeout 300 python bench.py --config $c $B --steps 250 --reps 5 > $O/bench_c${c}_250r5.json 2>/dev/null
  eval timeout 300 python bench.py --config $c $B --steps 1000 > $O/bench_c${c}_1000.json 2>/dev/null
done
S=";tile_order=1;tile_order=2;tile_order=11;tile_order=12;tile_order=13;tile_order=14;tile_order=15;tile_order=16"
timeout 900 python scripts/ab_knobs.py 3 "$S" 5 >> $O/ab_order.jsonl 2>> $O/ab_order.err
S=";tile_order=17;tile_order=21;tile_order=22;tile_order=23;tile_order=24;tile_order=25"
timeout 900 python scripts/ab_knobs.py 3 "$S" 5 >> $O/ab_order.jsonl 2>> $O/ab_order.err
eval timeout 300 python bench.py --config 3 $B --steps 300 > $O/bench_c3_300_end.json 2>/dev/null
echo done > $O/done.txt
