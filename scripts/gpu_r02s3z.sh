#!/bin/bash
# Smem gather first-wave bulk prefetch (knob gather_prefetch_waves).
O=gpurun_out/r02s3z
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "gather_launch_shapes or gather_random or gather_full" > $O/pytest.txt 2>&1
timeout 900 python scripts/ab_gather.py prefetch > $O/ab.jsonl 2> $O/ab.err
echo done > $O/done.txt
