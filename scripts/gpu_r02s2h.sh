#!/bin/bash
O=gpurun_out/r02s2h
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "tma" > $O/pytest_tma.txt 2>&1
timeout 900 python scripts/transpose_study.py > $O/transpose_study.jsonl 2> $O/transpose_study.err
echo done > $O/done.txt
