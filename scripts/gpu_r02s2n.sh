#!/bin/bash
O=gpurun_out/r02s2n
mkdir -p $O
timeout 900 python scripts/pattern_ceiling.py > $O/pattern_ceiling.jsonl 2> $O/pattern_ceiling.err
echo done > $O/done.txt
