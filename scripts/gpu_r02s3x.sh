#!/bin/bash
# Config 3: smaller granules (fewer registers per thread, higher occupancy).
O=gpurun_out/r02s3x
mkdir -p $O
S=";max_granule=8;max_granule=4;max_granule=8,smem_jit_minb=4;max_granule=8,smem_jit_minb=6;max_granule=4,smem_jit_minb=6"
timeout 1200 python scripts/ab_knobs.py 3 "$S" 5 >> $O/ab_granule.jsonl 2>> $O/ab.err
echo done > $O/done.txt
