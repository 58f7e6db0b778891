#!/bin/bash
# broadcast dedup (register zero columns, sliced layouts): GPU parity + smem
# instruction counts (tab:micro-broadcasting analogue); full GPU suite
O=gpurun_out/r02g
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "broadcast or sliced" > $O/pytest_bcast.txt 2>&1
timeout 900 python scripts/bcast_smem_counts.py > $O/bcast_smem_counts.json 2> $O/bcast_smem_counts.err
timeout 1500 python -m pytest tests -m gpu -q --durations=12 > $O/pytest_gpu.txt 2>&1
echo done > $O/done.txt
