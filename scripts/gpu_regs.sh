#!/bin/bash
# register-faithful path: in-kernel cycles (matrix vs vector) and full-size bench
OUT=gpurun_out/regs; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/regs_inkernel.py > $OUT/regs_inkernel.json 2> $OUT/regs_inkernel.err
B="--no-cpu-baseline --e2e-steps 0 --steps 300"
for c in 1 2; do
  timeout 200 python bench.py --config $c $B --path regs > $OUT/bench_regs_cfg$c.json 2> $OUT/bench_regs_cfg$c.err
  timeout 200 python bench.py --config $c $B --path regs --tune regs_matrix=0 > $OUT/bench_regsvec_cfg$c.json 2>/dev/null
  timeout 200 python bench.py --config $c $B > $OUT/bench_auto_cfg$c.json 2>/dev/null
done
