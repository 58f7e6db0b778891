#!/bin/bash
# Defaults with the first-wave PDL prefetch: GPU suite, default bench line,
# config 2 / 3 lines; gather PDL A/B (knob gather_pdl).
O=gpurun_out/r02s3g
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
B="--no-cpu-baseline --also '' --steps 300"
eval timeout 600 python bench.py --config 2 $B > $O/bench_cfg2.json 2> $O/bench_cfg2.err
eval timeout 600 python bench.py --config 3 $B > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python scripts/ab_gather.py pdl > $O/ab_gather_pdl.jsonl 2> $O/ab_gather.err
echo done > $O/done.txt
