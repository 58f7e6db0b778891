#!/bin/bash
# Bulk prologue prefetch on by default for the smem kernel: GPU suite, smoke,
# default line, config 2 / 3 / 6 lines; shuffle-kernel bulk prefetch A/B.
O=gpurun_out/r02s3bb
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
B="--no-cpu-baseline --also '' --steps 300"
for c in 3 2; do
  eval timeout 600 python bench.py --config $c $B > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 900 python scripts/ab_knobs.py 6 ";shuffle_prefetch_bulk=1" 5 >> $O/ab_shuffle_bulk.jsonl 2>> $O/ab.err
echo done > $O/done.txt
