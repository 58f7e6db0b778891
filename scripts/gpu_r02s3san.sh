#!/bin/bash
# compute-sanitizer over one small launch of every device path (round-2
# kernels included), each result checked against the oracle.
O=gpurun_out/r02s3san
mkdir -p $O
timeout 600 python scripts/sanitize_paths.py > $O/plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --target-processes all python scripts/sanitize_paths.py > $O/$t.txt 2>&1
done
echo done > $O/done.txt
