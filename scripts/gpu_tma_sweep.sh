#!/bin/bash
# TMA-fed path vs the smem path, knob sweep (stages, tile bytes, tiles per group)
OUT=gpurun_out/tma; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--no-cpu-baseline --e2e-steps 0 --steps 300"
for c in 3 5 2; do
  timeout 200 python bench.py --config $c $B > $OUT/smem_cfg$c.json 2>/dev/null
  for st in 2 3 4; do
    for tb in 8192 16384 32768; do
      timeout 200 python bench.py --config $c $B --path smem_tma --tune tma_stages=$st --tune tma_tile_bytes=$tb > $OUT/tma_cfg${c}_s${st}_t${tb}.json 2>$OUT/tma_cfg${c}_s${st}_t${tb}.err
    done
  done
  timeout 200 python bench.py --config $c $B --path smem_tma --tune tma_tpg=4 > $OUT/tma_cfg${c}_tpg4.json 2>/dev/null
  timeout 200 python bench.py --config $c $B --path smem_tma --tune tma_thread_bytes=128 > $OUT/tma_cfg${c}_tb128.json 2>/dev/null
done
