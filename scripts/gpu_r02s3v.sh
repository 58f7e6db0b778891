#!/bin/bash
# Chunk defaults by kind (32 MiB shards, 16 MiB instances / pitched): host
# tests and the e2e legs of configs 2 / 3 / 5.
O=gpurun_out/r02s3v
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "host" > $O/pytest.txt 2>&1
B="--no-cpu-baseline --also '' --ncu off --steps 50 --e2e-steps 8"
for c in 5 2 3; do
  eval timeout 300 python bench.py --config $c $B > $O/e2e_c$c.json 2>/dev/null
done
echo done > $O/done.txt
