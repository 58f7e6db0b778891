#!/bin/bash
# AUTO takes the shuffle exchange over the register permutation where it
# applies: GPU suite, classification rows, smoke.
O=gpurun_out/r02s3j
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python scripts/classify_bench.py > $O/classify.json 2> $O/classify_rows.jsonl
echo done > $O/done.txt
