#!/bin/bash
# In-situ bank conflicts: the compiled smem kernel with
# its global loads and / or stores removed (smem_jit_noload / _nostore: the
# identical STS / LDS schedule), ncu wavefronts per request; the TMA kernels'
# readers (no LDG at all) on the same configs.
O=gpurun_out/r02s2c
mkdir -p $O
B="--no-cpu-baseline --e2e-steps 0 --also '' --steps 200 --ncu on"
for c in 3 2 5; do
  eval timeout 300 python bench.py --config $c $B > $O/bench_c${c}.json 2> $O/bench_c${c}.err
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_noload=1 > $O/bench_c${c}_noload.json 2> $O/bench_c${c}_noload.err
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_nostore=1 > $O/bench_c${c}_nostore.json 2> $O/bench_c${c}_nostore.err
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_noload=1 --tune smem_jit_nostore=1 > $O/bench_c${c}_nols.json 2> $O/bench_c${c}_nols.err
  for p in smem_tma smem_tma_store; do
    eval timeout 300 python bench.py --config $c --path $p $B > $O/bench_c${c}_$p.json 2> $O/bench_c${c}_$p.err
  done
done
echo done > $O/done.txt
