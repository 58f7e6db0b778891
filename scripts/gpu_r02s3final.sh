#!/bin/bash
# Round 2 (session 3) consolidated run on the committed head: smoke, GPU suite, the default
# bench line, its ncu launch list, one ncu --set full capture of the dominant
# kernel, the reference arm, cfg4full / upcast / cfg6 lines, knob A/B on cfg5.
O=gpurun_out/${FINAL_TAG:-r02s3final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --ncu off > $O/bench_under_ncu.log 2>&1
export LL_JIT_SOURCE_DIR=$PWD/$O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ll_smem_hbm -c 1 -o $O/cfg5_smem_full \
  python bench.py --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu_full.log 2>&1
unset LL_JIT_SOURCE_DIR
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
B="--no-cpu-baseline --also '' --steps 300"
eval timeout 600 python bench.py --config 4full $B > $O/bench_cfg4full.json 2> $O/bench_cfg4full.err
eval timeout 600 python bench.py --config 6 $B > $O/bench_cfg6.json 2> $O/bench_cfg6.err
eval timeout 600 python bench.py --config 5 --upcast $B > $O/bench_upcast.json 2> $O/bench_upcast.err
timeout 900 python scripts/ab_paths.py 3 > $O/ab_paths.jsonl 2> $O/ab_paths.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_timed.csv \
  python bench.py --steps 20 --warmup 3 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' --reps 2 > $O/bench_timed_under_ncu.log 2>&1
export LL_JIT_SOURCE_DIR=$PWD/$O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ll_gather_smem -c 1 -o $O/cfg4_gather_full \
  python bench.py --config 4 --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu_full_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ll_shfl_hbm -c 1 -o $O/cfg6_shfl_full \
  python bench.py --config 6 --steps 2 --warmup 1 --reps 1 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' > $O/ncu_full_cfg6.log 2>&1
unset LL_JIT_SOURCE_DIR
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; done
echo done > $O/done.txt
