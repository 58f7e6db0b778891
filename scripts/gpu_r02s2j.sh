#!/bin/bash
# TMA-load 256-bit stores (config 2): parity, interleaved A/B; the sanitizer
# workload to the end; a launch list of the timed region alone.
O=gpurun_out/r02s2j
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "tma" > $O/pytest_tma.txt 2>&1
timeout 900 python scripts/ab_paths.py 3 > $O/ab_paths.jsonl 2> $O/ab_paths.err
timeout 600 python scripts/sanitize_paths.py > $O/plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --target-processes all python scripts/sanitize_paths.py > $O/$t.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_timed.csv \
  python bench.py --steps 20 --warmup 3 --ncu off --no-cpu-baseline --e2e-steps 0 --also '' --reps 2 > $O/bench_under_ncu.log 2>&1
echo done > $O/done.txt
