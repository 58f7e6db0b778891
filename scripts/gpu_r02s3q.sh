#!/bin/bash
# ll_convert_host_shard: parity, and the two-rank flow (gloo, one GPU) whose
# e2e leg now runs it per rank.
O=gpurun_out/r02s3q
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "host" > $O/pytest.txt 2>&1
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_gloo2.json 2> $O/bench_gloo2.err
echo done > $O/done.txt
