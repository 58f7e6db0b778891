#!/bin/bash
# Second-wave prefetch in the shuffle kernel (knob shuffle_prefetch_waves), config 6.
O=gpurun_out/r02s3y
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "shuffle_kernel_pdl" > $O/pytest.txt 2>&1
timeout 900 python scripts/ab_knobs.py 6 ";shuffle_prefetch_waves=2;shuffle_prefetch_waves=3" 7 >> $O/ab.jsonl 2>> $O/ab.err
echo done > $O/done.txt
