#!/bin/bash
# TMA load + store path: parity tests, then a knob sweep vs the smem path
OUT=gpurun_out/tmas; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tma" > $OUT/pytest_tma.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --steps 300"
for c in 3 2 5; do
  timeout 200 python bench.py --config $c $B > $OUT/smem_cfg$c.json 2>/dev/null
  for st in 2 3; do for rb in 128 256; do
    timeout 200 python bench.py --config $c $B --path smem_tma_store --tune tma_stages=$st --tune tma_run_bytes=$rb > $OUT/tmas_cfg${c}_s${st}_rb${rb}.json 2>$OUT/tmas_cfg${c}_s${st}_rb${rb}.err
  done; done
  timeout 200 python bench.py --config $c $B --path smem_tma_store --tune tma_tpg=2 > $OUT/tmas_cfg${c}_tpg2.json 2>/dev/null
  timeout 200 python bench.py --config $c $B --path smem_tma_store --tune tma_thread_bytes=128 > $OUT/tmas_cfg${c}_tb128.json 2>/dev/null
done
