#!/bin/bash
# Non-persistent compiled TMA kernels (tmaj_tpc tiles per group and CTA,
# several CTAs per SM so the next launch fills SMs while one drains);
# regperm one-pass default; classification bench.
O=gpurun_out/r02s2f
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "tma or permutation" > $O/pytest.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for c in 2 3 5 6; do
  for p in smem_tma smem_tma_store; do
    for v in "2 2 2" "4 2 2" "8 2 2" "4 2 3" "8 2 3" "4 1 3" "16 1 3" "2 3 2" "4 3 2"; do
      set -- $v
      eval timeout 300 python bench.py --config $c --path $p $B --tune tmaj_tpc=$1 --tune tmaj_cps=$2 --tune tmaj_stages=$3 > $O/bench_c${c}_${p}_t$1_c$2_s$3.json 2>/dev/null
    done
  done
done
timeout 600 python scripts/regperm_sweep.py > $O/regperm_sweep.jsonl 2> $O/regperm_sweep.err
timeout 600 python scripts/classify_bench.py > $O/classify.json 2> $O/classify.err
echo done > $O/done.txt
