#!/bin/bash
O=gpurun_out/r02s2r
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "permutation or broadcast or sliced or cfg6" > $O/pytest.txt 2>&1
timeout 900 python scripts/classify_bench.py > $O/classify.json 2> $O/classify_rows.jsonl
echo done > $O/done.txt
