#!/bin/bash
# One GPU session: probe, build check, smoke, gpu tests, bench, launch list.
set -x
mkdir -p gpurun_out
{ nvidia-smi; nproc; python -c "import torch;p=torch.cuda.get_device_properties(0);print(p)"; } > gpurun_out/probe.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in 3 4 5 1; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
