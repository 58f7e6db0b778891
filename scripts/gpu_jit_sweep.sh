#!/bin/bash
# plan-compiled smem kernel: register cap (resident CTAs) x tiles per group
OUT=gpurun_out/jitsw; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--no-cpu-baseline --e2e-steps 0 --steps 300"
for c in 3 2 5; do
  for mb in 2 3 4 5; do for tpg in 1 2; do
    timeout 200 python bench.py --config $c $B --tune smem_jit_minb=$mb --tune smem_jit_tpg=$tpg > $OUT/cfg${c}_minb${mb}_tpg${tpg}.json 2>/dev/null
  done; done
done
