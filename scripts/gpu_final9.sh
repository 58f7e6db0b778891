#!/bin/bash
# Consolidated measurement (round 1, last: every default as committed, after the
# gather and host-pipeline changes): tests, smoke, bench per config and per alternative path,
# reference arm, in-kernel cycles, ncu launch lists and full captures.
O=gpurun_out/final9
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
for c in 3 4 5 1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 600 python bench.py --config 5 --upcast --no-cpu-baseline > $O/bench_cfg5_upcast.json 2> $O/bench_cfg5_upcast.err
B="--no-cpu-baseline --e2e-steps 0"
timeout 300 python bench.py --config 3 $B --path smem_tma > $O/bench_cfg3_tma.json 2>/dev/null
timeout 300 python bench.py --config 5 $B --path smem_tma > $O/bench_cfg5_tma.json 2>/dev/null
timeout 300 python bench.py --config 2 $B --path smem_tma > $O/bench_cfg2_tma.json 2>/dev/null
timeout 300 python bench.py --config 2 $B --path regs > $O/bench_cfg2_regs.json 2>/dev/null
timeout 300 python bench.py --config 1 $B --path regs > $O/bench_cfg1_regs.json 2>/dev/null
timeout 300 python bench.py --config 4 $B --path shuffle > $O/bench_cfg4_shuffle.json 2>/dev/null
for c in 2 3 5; do timeout 300 python bench.py --config $c $B --tune smem_jit=0 > $O/bench_cfg${c}_generic.json 2>/dev/null; done
for c in 2 5; do timeout 300 python bench.py --config $c $B --path shuffle > $O/bench_cfg${c}_shfl.json 2>/dev/null; done
for c in 2 3 5; do timeout 300 python bench.py --config $c $B --path smem_tma_store --tune tma_stages=2 > $O/bench_cfg${c}_tmas.json 2>/dev/null; done
timeout 300 python scripts/regs_inkernel.py > $O/regs_inkernel.json 2> $O/regs_inkernel.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err
# launch lists (cold, serialised: shares only)
for c in 2 3 4 5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"convert|gather|ll_" -c 20 --csv --log-file $O/launches_cfg$c.csv python bench.py --config $c --steps 20 --warmup 5 $B > /dev/null 2>&1
done
# full captures of the dominant kernels
cap() { # name, kernel regex, bench args
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 5 -c 1 -o $O/prof_$1 python bench.py --steps 10 --warmup 5 $B $3 > $O/ncu_$1.log 2>&1
}
cap cfg2_jit ll_smem_hbm "--config 2"
cap cfg2 convert_smem "--config 2 --tune smem_jit=0"
cap cfg5_shfl ll_shfl_hbm "--config 5 --path shuffle"
cap cfg3_jit ll_smem_hbm "--config 3"
cap cfg4 gather_direct "--config 4"
cap cfg4_shfl gather_shuffle "--config 4 --path shuffle"
cap cfg5_jit ll_smem_hbm "--config 5"
cap cfg5_upcast_jit ll_upcast_hbm "--config 5 --upcast"
cap cfg5_upcast convert_smem "--config 5 --upcast --tune upcast_jit=0"
cap cfg3_tma convert_tma "--config 3 --path smem_tma"
cap cfg5_tma convert_tma "--config 5 --path smem_tma"
cap cfg2_regs convert_regs "--config 2 --path regs"
cap cfg3_tmas convert_tma_store "--config 3 --path smem_tma_store"
timeout 300 ncu --set full --clock-control none -k regex:ll_regs_shfl -c 1 -o $O/prof_cfg2w_regs_shfl python scripts/regs_one.py 2w shfl 64 > $O/ncu_cfg2w_regs_shfl.log 2>&1
# keep the copy-back under 64 MiB: summaries + raw csv pages, then drop the reports
python scripts/ncu_summary.py $O/prof_*.ncu-rep > $O/ncu_summary.json 2> $O/ncu_summary.err
for r in $O/prof_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
done
rm -f $O/prof_*.ncu-rep
