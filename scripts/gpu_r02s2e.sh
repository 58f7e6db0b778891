#!/bin/bash
# regperm variants; config-3 LDG-path sweep; ncu --set full of the compiled
# TMA kernel (cfg2, load + store variants) and of the cfg3 default kernel.
O=gpurun_out/r02s2e
mkdir -p $O
timeout 600 python scripts/regperm_sweep.py > $O/regperm_sweep.jsonl 2> $O/regperm_sweep.err
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
eval timeout 300 python bench.py --config 3 $B > $O/sweep3_default.json 2>/dev/null
for t in "vec32=1" "tile_order=1" "tile_order=2" "run_bytes_dst=128" "run_bytes_dst=256" "thread_bytes=128" "thread_bytes=32" "smem_jit_depth=2" "smem_jit_tpg=2" "smem_jit_minb=2" "smem_jit_minb=3" "auto_asym=0" "run_bytes=512" "run_bytes_src=512" "smem_jit_single=1"; do
  eval timeout 300 python bench.py --config 3 $B --tune $t > $O/sweep3_$t.json 2>/dev/null
done
N="ncu --set full --clock-control none --import-source on -c 1"
B1="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 2 --warmup 1 --reps 1"
export LL_JIT_SOURCE_DIR=$PWD/$O
eval timeout 600 $N -k regex:ll_tma_hbm -o $O/tma_cfg2_load python bench.py --config 2 --path smem_tma $B1 > $O/ncu_tma2.log 2>&1
eval timeout 600 $N -k regex:ll_tma_hbm -o $O/tma_cfg2_store python bench.py --config 2 --path smem_tma_store $B1 > $O/ncu_tma2s.log 2>&1
eval timeout 600 $N -k regex:ll_smem_hbm -o $O/smem_cfg3 python bench.py --config 3 $B1 > $O/ncu_smem3.log 2>&1
eval timeout 600 $N -k regex:ll_tma_hbm -o $O/tma_cfg3_store python bench.py --config 3 --path smem_tma_store $B1 > $O/ncu_tma3s.log 2>&1
echo done > $O/done.txt
