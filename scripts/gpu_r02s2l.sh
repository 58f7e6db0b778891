#!/bin/bash
O=gpurun_out/r02s2l
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "gather" > $O/pytest_gather.txt 2>&1
timeout 900 python scripts/ab_gather.py > $O/ab_gather.jsonl 2> $O/ab_gather.err
echo done > $O/done.txt
