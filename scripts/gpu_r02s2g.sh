#!/bin/bash
# Defaults after the TMA / regperm changes: TMA + permutation parity, then the
# interleaved path A/B on every config, then the full suite.
O=gpurun_out/r02s2g
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "tma or permutation or b8" > $O/pytest_new.txt 2>&1
timeout 1500 python scripts/ab_paths.py 3 > $O/ab_paths.jsonl 2> $O/ab_paths.err
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
echo done > $O/done.txt
