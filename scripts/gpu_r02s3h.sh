#!/bin/bash
# Gather PDL + AUTO smem gather, shuffle-kernel PDL (knob shuffle_pdl),
# regperm first-wave prefetch: GPU suite, A/Bs, config 4 / 4full lines.
O=gpurun_out/r02s3h
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python scripts/ab_gather.py pdl > $O/ab_gather_pdl.jsonl 2> $O/ab_gather.err
for c in 6; do
  timeout 600 python scripts/ab_knobs.py $c ";shuffle_pdl=1" 7 >> $O/ab_shuffle_pdl.jsonl 2>> $O/ab.err
done
timeout 900 python scripts/ab_regperm_prefetch.py > $O/ab_regperm.jsonl 2>> $O/ab.err
B="--no-cpu-baseline --also '' --steps 300"
eval timeout 600 python bench.py --config 4 $B > $O/bench_cfg4.json 2> $O/bench_cfg4.err
eval timeout 600 python bench.py --config 4full $B > $O/bench_cfg4full.json 2> $O/bench_cfg4full.err
echo done > $O/done.txt
