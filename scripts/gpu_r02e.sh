#!/bin/bash
# vec32 (256-bit LDG/STG) A/B and the in-situ bank-conflict experiment
# (smem_jit_noload: the same STS/LDS schedule with register-made data).
O=gpurun_out/r02e
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "vec32 or configs_small or random_pairs" > $O/pytest.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --also '' --steps 300"
for c in 2 3 5; do
  eval timeout 300 python bench.py --config $c $B > $O/bench_cfg${c}.json 2> $O/bench_cfg${c}.err
  eval timeout 300 python bench.py --config $c $B --tune vec32=1 > $O/bench_cfg${c}_vec32.json 2> $O/bench_cfg${c}_vec32.err
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_noload=1 --ncu on > $O/bench_cfg${c}_noload.json 2> $O/bench_cfg${c}_noload.err
done
echo done > $O/done.txt
