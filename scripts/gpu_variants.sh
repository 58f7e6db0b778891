#!/bin/bash
# Build variants (LL_NVCC_EXTRA flag sets, ';'-separated in VARIANTS) and bench
# each on CONFIGS (default "2 3 5"); the default build is rebuilt at the end.
# Optional: BENCH_ARGS (extra bench.py flags), OUT (subdir of gpurun_out).
OUT=gpurun_out/${OUT:-variants}
mkdir -p $OUT
CONFIGS=${CONFIGS:-"2 3 5"}
python -c "import __graft_entry__ as g; g.build()"
IFS=';' read -ra VS <<< "${VARIANTS}"
for rep in 1 2; do
  for c in $CONFIGS; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 $BENCH_ARGS > $OUT/default_cfg${c}_$rep.json 2>/dev/null
  done
  for v in "${VS[@]}"; do
    name=$(echo "$v" | tr -d ' =-')
    LL_NVCC_EXTRA="$v" python paper_2505_23819_b200/build.py --force > /dev/null 2>&1
    for c in $CONFIGS; do
      timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 $BENCH_ARGS > $OUT/${name}_cfg${c}_$rep.json 2>/dev/null
    done
  done
  python paper_2505_23819_b200/build.py --force > /dev/null 2>&1
done
if [ -d _ab_old ]; then
  for c in $CONFIGS; do (cd _ab_old && timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0) > $OUT/old_cfg${c}.json 2>/dev/null; done
fi
