#!/bin/bash
# Write-heavy ceilings for the fused upcast (reads 1 B, writes 4 B).
O=gpurun_out/r02s3s
mkdir -p $O
timeout 600 python scripts/write_ceiling.py > $O/write_ceiling.jsonl 2> $O/write_ceiling.err
B="--no-cpu-baseline --also '' --steps 100 --ncu off"
eval timeout 600 python bench.py --config 5 --upcast $B > $O/bench_upcast.json 2> $O/bench_upcast.err
echo done > $O/done.txt
