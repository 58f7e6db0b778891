#!/bin/bash
# Shuffle kernel bulk prefetch on by default: GPU suite, smoke, config 6 / 3 / default lines.
O=gpurun_out/r02s3cc
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
B="--no-cpu-baseline --also '' --steps 300"
for c in 6 3; do
  eval timeout 600 python bench.py --config $c $B > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo done > $O/done.txt
