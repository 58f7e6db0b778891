#!/bin/bash
# Gather end to end: chunk size x staging (config 4).
O=gpurun_out/r02s3u
mkdir -p $O
B="--no-cpu-baseline --also '' --ncu off --steps 50 --e2e-steps 8"
for ch in 16 32 8; do
  for sm in 32 64; do
    eval timeout 300 python bench.py --config 4 $B --tune host_chunk_mb=$ch --e2e-gather-scratch-mb $sm > "$O/e2e_c${ch}_s${sm}.json" 2>/dev/null
  done
done
echo done > $O/done.txt
