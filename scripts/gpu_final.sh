#!/bin/bash
# consolidated round measurement: tests, smoke, bench per config, ncu per config
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
for c in 3 4 5 1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/final/bench_cfg$c.json 2> gpurun_out/final/bench_cfg$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
for c in 2 3 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"convert_smem|gather" -s 5 -c 1 -o gpurun_out/final/prof_cfg$c python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/final/ncu_cfg$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"convert|gather" -c 20 --csv --log-file gpurun_out/final/launches_cfg$c.csv python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
