#!/bin/bash
# Diagonal tile order (knob tile_xor) on config 3 (and 2 / 5), parity tests,
# the two-rank gloo flow on one GPU.
O=gpurun_out/r02s3l
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "hint_and_order or tile_xor" > $O/pytest.txt 2>&1
S=";tile_xor=2;tile_xor=4;tile_xor=6;tile_xor=4,tile_xor_skip=0;tile_xor=6,tile_xor_skip=2"
timeout 900 python scripts/ab_knobs.py 3 "$S" 5 >> $O/ab_xor.jsonl 2>> $O/ab.err
timeout 900 python scripts/ab_knobs.py 2 ";tile_xor=4;tile_xor=6" 5 >> $O/ab_xor.jsonl 2>> $O/ab.err
timeout 900 python scripts/ab_knobs.py 5 ";tile_xor=4;tile_xor=6" 5 >> $O/ab_xor.jsonl 2>> $O/ab.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_gloo2.json 2> $O/bench_gloo2.err
echo done > $O/done.txt
