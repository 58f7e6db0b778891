#!/bin/bash
# ncu evidence on the final head: launch list of the default command and of
# the timed region, ncu --set full of the config-5 and config-3 kernels.
O=gpurun_out/r02s3dd
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --ncu off > $O/bench_under_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_timed.csv \
  python bench.py --steps 20 --warmup 3 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' --reps 2 > $O/bench_timed_under_ncu.log 2>&1
export LL_JIT_SOURCE_DIR=$PWD/$O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ll_smem_hbm -c 1 -o $O/cfg5_smem_full \
  python bench.py --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ll_smem_hbm -c 1 -o $O/cfg3_smem_full \
  python bench.py --config 3 --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu3.log 2>&1
unset LL_JIT_SOURCE_DIR
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; done
echo done > $O/done.txt
