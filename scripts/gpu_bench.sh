#!/bin/bash
mkdir -p gpurun_out/bench
python -c "import __graft_entry__ as g; g.build()"
for c in ${CFGS:-2 3 4 5 1}; do timeout 600 python bench.py --config $c ${EXTRA} > gpurun_out/bench/bench_cfg$c.json 2> gpurun_out/bench/bench_cfg$c.err; done
