#!/bin/bash
# bench + one ncu --set full capture of the fused mxfp4 upcast kernel (config 5)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --config 5 --upcast --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_upcast.json 2> gpurun_out/bench_upcast.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"convert_smem" -s 5 -c 1 -o gpurun_out/prof_upcast${TAG} python bench.py --config 5 --upcast --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-graph > gpurun_out/ncu_upcast.log 2>&1
