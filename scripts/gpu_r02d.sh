#!/bin/bash
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k gather > $O/pytest_gather.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 200"
for p in generic shuffle smem; do eval timeout 300 python bench.py --config 4 --path $p $B > $O/bench_cfg4_$p.json 2> $O/bench_cfg4_$p.err; done
for mu in 2 8; do eval timeout 300 python bench.py --config 4 --path shuffle --tune gather_shfl_mu=$mu $B > $O/bench_cfg4_shuffle_mu$mu.json 2>/dev/null; done
for x in 1 2; do eval timeout 300 python bench.py --config 4 --path smem --tune gather_cta_extra=$x $B > $O/bench_cfg4_smem_x$x.json 2>/dev/null; done
for p in generic smem; do eval timeout 300 python bench.py --config 4full --path $p $B > $O/bench_cfg4full_$p.json 2> $O/bench_cfg4full_$p.err; done
timeout 300 python scripts/gather_inkernel.py > $O/gather_inkernel.json 2> $O/gather_inkernel.err
echo done > $O/done.txt
