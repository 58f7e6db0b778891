#!/bin/bash
# upcast kernel: default build vs LL_NVCC_EXTRA variants (bench config 5 --upcast).
# VARIANTS: ';'-separated nvcc flag sets.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --config 5 --upcast --no-cpu-baseline --e2e-steps 0 > gpurun_out/up_default.json 2>&1
IFS=';' read -ra VS <<< "${VARIANTS:--DLL_UP_MINB=3}"
for v in "${VS[@]}"; do
  name=$(echo "$v" | tr -d ' =-')
  LL_NVCC_EXTRA="$v" python paper_2505_23819_b200/build.py --force > /dev/null
  timeout 300 python bench.py --config 5 --upcast --no-cpu-baseline --e2e-steps 0 > "gpurun_out/up_$name.json" 2>&1
done
python paper_2505_23819_b200/build.py --force > /dev/null
