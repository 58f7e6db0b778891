#!/bin/bash
# A/B: an older worktree (_ab_old) vs HEAD, same box, alternating
mkdir -p gpurun_out/ab
for c in 2 3 5; do
  for rep in 1 2; do
    (cd _ab_old && timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0) > gpurun_out/ab/old_cfg${c}_$rep.json 2>/dev/null
    timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab/new_cfg${c}_$rep.json 2>/dev/null
  done
done
