#!/bin/bash
# ncu captures (one launch each) of the dominant kernel of every bench config
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for c in ${CFGS:-2 3 4 5}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"convert_smem|gather" -s 5 -c 1 -o gpurun_out/prof_cfg$c python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_cfg$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"convert|gather" -c 20 --csv --log-file gpurun_out/launches_cfg$c.csv python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
