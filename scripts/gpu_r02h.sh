#!/bin/bash
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "broadcast or sliced or permutation" > $O/pytest_new.txt 2>&1
timeout 900 python scripts/classify_bench.py > $O/classify.json 2> $O/classify.err
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
echo done > $O/done.txt
