#!/bin/bash
# Session 3 first run: head check (smoke, GPU suite, default bench line).
O=gpurun_out/r02s3a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
B="--no-cpu-baseline --also '' --steps 300"
eval timeout 600 python bench.py --config 3 $B > $O/bench_cfg3.json 2> $O/bench_cfg3.err
echo done > $O/done.txt
