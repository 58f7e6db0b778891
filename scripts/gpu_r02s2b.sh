#!/bin/bash
# Warp-specialised TMA kernels compiled per plan: parity, then path x knob
# sweep on configs 2 / 3 / 5 (CUDA-graph bench, no ncu), ncu of cfg3 TMA.
O=gpurun_out/r02s2b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "tma" > $O/pytest_tma.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for c in 3 2 5; do
  for p in smem_tma smem_tma_store; do
    eval timeout 300 python bench.py --config $c --path $p $B > $O/bench_c${c}_${p}.json 2> $O/bench_c${c}_${p}.err
    for t in "tmaj_cps=2" "tmaj_stages=3" "tmaj_stages=4" "pdl=0" "tmaj_k=1"; do
      eval timeout 300 python bench.py --config $c --path $p $B --tune $t > $O/bench_c${c}_${p}_$t.json 2>/dev/null
    done
  done
  eval timeout 300 python bench.py --config $c $B > $O/bench_c${c}_auto.json 2> $O/bench_c${c}_auto.err
done

# config 6 (pre-shuffle): parity + default line and path sweep
timeout 900 python -m pytest tests -m gpu -q -k "cfg6" > $O/pytest_cfg6.txt 2>&1
for p in auto smem shuffle smem_tma smem_tma_store; do
  eval timeout 300 python bench.py --config 6 --path $p $B > $O/bench_c6_$p.json 2> $O/bench_c6_$p.err
done
echo done > $O/done.txt
