#!/bin/bash
# Last check of the session-3 head: smoke, GPU suite, default line, config
# 2 / 3 / 4 / 4full / 6 lines.
O=gpurun_out/r02s3fin
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
B="--no-cpu-baseline --also '' --steps 300"
for c in 2 3 4 4full 6; do
  eval timeout 600 python bench.py --config $c $B > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
echo done > $O/done.txt
