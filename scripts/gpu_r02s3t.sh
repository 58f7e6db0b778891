#!/bin/bash
# Host-buffer binding checks on the GPU: host tests, default bench line.
O=gpurun_out/r02s3t
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "host" > $O/pytest.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo done > $O/done.txt
