#!/bin/bash
# Round 2, session 2, first pass on the current head: smoke, the whole GPU
# suite, the default bench line (ncu subprocess), the multi-rank flow (gloo,
# 2 ranks on one GPU), cfg4full / upcast lines, the reference arm, the
# classification / broadcast / gather studies.
O=gpurun_out/r02s2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_gloo2.json 2> $O/bench_gloo2.err
timeout 600 python bench.py --config 4full --steps 200 --no-cpu-baseline --also "" > $O/bench_cfg4full.json 2> $O/bench_cfg4full.err
timeout 600 python bench.py --config 5 --upcast --steps 100 --no-cpu-baseline --also "" > $O/bench_upcast.json 2> $O/bench_upcast.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python scripts/classify_bench.py > $O/classify.json 2> $O/classify.err
timeout 900 python scripts/bcast_smem_counts.py > $O/bcast_smem_counts.json 2> $O/bcast_smem_counts.err
timeout 300 python scripts/gather_inkernel.py > $O/gather_inkernel.json 2> $O/gather_inkernel.err
echo done > $O/done.txt
