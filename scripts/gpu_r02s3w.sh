#!/bin/bash
# ncu --set full of config 3's kernel (the one VERDICT r1 named) on the final head.
O=gpurun_out/r02s3w
mkdir -p $O
export LL_JIT_SOURCE_DIR=$PWD/$O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ll_smem_hbm -c 1 -o $O/cfg3_smem_full \
  python bench.py --config 3 --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu.log 2>&1
unset LL_JIT_SOURCE_DIR
ncu -i $O/cfg3_smem_full.ncu-rep --page raw --csv > $O/cfg3_smem_full_raw.csv 2>/dev/null
ncu -i $O/cfg3_smem_full.ncu-rep --page details --csv > $O/cfg3_smem_full_details.csv 2>/dev/null
ncu -i $O/cfg3_smem_full.ncu-rep --page source --csv --print-source sass > $O/cfg3_smem_full_source.csv 2>/dev/null
echo done > $O/done.txt
