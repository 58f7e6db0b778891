#!/bin/bash
# build, gpu tests, sweep, ncu of the cfg2 kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python scripts/sweep.py --steps 100 --knobs "${KNOBS:-tpg=0,2,4;pipe=0,1}" --paths "${PATHS:-smem,smem_noswizzle}" > gpurun_out/sweep.log 2>&1
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:convert_smem -s 5 -c 1 -o gpurun_out/prof_cfg${NCU} python bench.py --config ${NCU} --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu.log 2>&1
fi
