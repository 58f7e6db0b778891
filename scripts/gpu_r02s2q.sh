#!/bin/bash
O=gpurun_out/r02s2q
mkdir -p $O
timeout 300 python -m pytest tests -m gpu -q -x -k "permutation" > $O/pytest.txt 2>&1
timeout 900 python scripts/regperm_sweep.py > $O/regperm_sweep.jsonl 2> $O/regperm_sweep.err
echo done > $O/done.txt
