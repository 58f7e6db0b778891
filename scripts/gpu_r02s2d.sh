#!/bin/bash
# TMA kernels with the proxy fence: full-size diagnosis, perf sweep
# (stages x CTAs per SM), the GPU suite; AUTO's small-granule shuffle rule
# (config 6); in-situ bank-conflict experiment (scripts/gpu_r02s2c.sh).
O=gpurun_out/r02s2d
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python scripts/tma_diag.py > $O/tma_diag.jsonl 2> $O/tma_diag.err
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for c in 3 2 5 6; do
  eval timeout 300 python bench.py --config $c $B > $O/bench_c${c}_auto.json 2> $O/bench_c${c}_auto.err
  for p in smem_tma smem_tma_store; do
    for st in 2 3 4 6; do
      for cps in 1 2; do
        eval timeout 300 python bench.py --config $c --path $p $B --tune tmaj_stages=$st --tune tmaj_cps=$cps > $O/bench_c${c}_${p}_s${st}_c${cps}.json 2>/dev/null
      done
    done
  done
done
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
bash scripts/gpu_r02s2c.sh
echo done > $O/done.txt
