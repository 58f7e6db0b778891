#!/bin/bash
O=gpurun_out/r02s2p
mkdir -p $O
timeout 900 python scripts/shard_projection.py > $O/shard_projection.jsonl 2> $O/shard_projection.err
echo done > $O/done.txt
