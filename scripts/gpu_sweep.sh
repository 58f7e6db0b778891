#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python scripts/sweep.py --steps 100 > gpurun_out/sweep.log 2>&1
# ncu: launch list of the convert kernel only, then one full capture
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"convert|gather" -c 30 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:convert_smem -s 5 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_cfg2.log 2>&1
