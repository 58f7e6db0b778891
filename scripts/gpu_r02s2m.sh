#!/bin/bash
O=gpurun_out/r02s2m
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "gather" > $O/pytest_gather.txt 2>&1
timeout 900 python scripts/ab_gather.py > $O/ab_gather.jsonl 2> $O/ab_gather.err
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 100"
for t in 4 1 2 8; do
  eval timeout 300 python bench.py --config 5 --upcast $B --tune upcast_jit_tpg=$t > $O/upcast_tpg$t.json 2>/dev/null
done
echo done > $O/done.txt
