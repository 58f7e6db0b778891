#!/bin/bash
# Round 2, first pass: GPU suite (whole-buffer full-size parity), smoke, the
# default bench line (cfg5 + also 2/3/4, ncu subprocess), the multi-rank flow
# (2 ranks on one GPU, gloo), the full-axis gather, the upcast e2e fix, and
# the reference arm.
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_gloo2.json 2> $O/bench_gloo2.err
timeout 600 python bench.py --config 4full --steps 200 --no-cpu-baseline --also "" > $O/bench_cfg4full.json 2> $O/bench_cfg4full.err
timeout 600 python bench.py --config 5 --upcast --steps 100 --no-cpu-baseline > $O/bench_upcast.json 2> $O/bench_upcast.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
echo done > $O/done.txt
