#!/bin/bash
# compute-sanitizer over one small launch of every device path
O=gpurun_out/sanitize; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths.py > $O/$tool.txt 2>&1
  echo "exit=$?" >> $O/$tool.txt
done
