#!/bin/bash
# cfg3 transpose: tile order x tiles per group x pipelining (after the register cap)
OUT=gpurun_out/cfg3sw; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--config 3 --no-cpu-baseline --e2e-steps 0 --steps 200"
for to in 0 1 2; do for tpg in 1 2 4 0; do for pipe in 1 0; do
  timeout 120 python bench.py $B --tune tile_order=$to --tune tpg=$tpg --tune pipe=$pipe > $OUT/to${to}_tpg${tpg}_p${pipe}.json 2>/dev/null
done; done; done
for rb in 128 512; do timeout 120 python bench.py $B --tune run_bytes=$rb > $OUT/rb$rb.json 2>/dev/null; done
for tb in 32 128; do timeout 120 python bench.py $B --tune thread_bytes=$tb > $OUT/tb$tb.json 2>/dev/null; done
