#!/bin/bash
# programmatic dependent launch on the plan-compiled smem kernel: on / off
OUT=gpurun_out/pdl; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "configs_small or random_pairs or ragged or shards" > $OUT/pytest.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --steps 500"
for rep in 1 2; do for c in 2 3 5; do
  timeout 200 python bench.py --config $c $B > $OUT/cfg${c}_pdl_$rep.json 2>/dev/null
  timeout 200 python bench.py --config $c $B --tune pdl=0 > $OUT/cfg${c}_nopdl_$rep.json 2>/dev/null
done; done
timeout 200 python bench.py --config 2 $B --no-graph > $OUT/cfg2_pdl_nograph.json 2>/dev/null
timeout 200 python bench.py --config 2 $B --no-graph --tune pdl=0 > $OUT/cfg2_nopdl_nograph.json 2>/dev/null
