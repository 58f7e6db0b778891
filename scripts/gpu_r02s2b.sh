#!/bin/bash
# Session 2, second pass: the warp-specialised TMA kernels (parity, then path
# x knob sweep on configs 2 / 3 / 5 / 6), the .b8 matrix tiles on the
# register-faithful path (parity + in-kernel cycles), the regperm kernel
# with several chunks per thread (classification bench), config 6.
O=gpurun_out/r02s2b
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "tma or b8 or cfg6 or permutation" > $O/pytest_new.txt 2>&1
timeout 600 python scripts/b8_inkernel.py > $O/b8_inkernel.json 2> $O/b8_inkernel.err
timeout 600 python scripts/classify_bench.py > $O/classify.json 2> $O/classify.err
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for c in 3 2 5 6; do
  eval timeout 300 python bench.py --config $c $B > $O/bench_c${c}_auto.json 2> $O/bench_c${c}_auto.err
  for p in smem_tma smem_tma_store; do
    eval timeout 300 python bench.py --config $c --path $p $B > $O/bench_c${c}_${p}.json 2> $O/bench_c${c}_${p}.err
    for t in "tmaj_cps=2" "tmaj_stages=3" "tmaj_stages=4" "pdl=0" "tmaj_k=1" "tma_jit=0"; do
      eval timeout 300 python bench.py --config $c --path $p $B --tune $t > $O/bench_c${c}_${p}_$t.json 2>/dev/null
    done
  done
done
eval timeout 300 python bench.py --config 6 --path shuffle $B > $O/bench_c6_shuffle.json 2> $O/bench_c6_shuffle.err
echo done > $O/done.txt
