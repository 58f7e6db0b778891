#!/bin/bash
# End-to-end chunking on config 5 (host_chunk_mb x host_slots) against the
# PCIe ceiling (scripts/pcie_probe.py).
O=gpurun_out/r02s3n
mkdir -p $O
timeout 300 python scripts/pcie_probe.py > $O/pcie_probe.json 2> $O/pcie_probe.err
B="--no-cpu-baseline --also '' --ncu off --steps 50"
for v in "host_chunk_mb=16" "host_chunk_mb=8" "host_chunk_mb=4" "host_chunk_mb=32" "host_chunk_mb=8,host_slots=3" "host_chunk_mb=4,host_slots=4" "host_chunk_mb=16,host_slots=3"; do
  T=""; for kv in ${v//,/ }; do T="$T --tune $kv"; done
  eval timeout 300 python bench.py --config 5 $B $T > "$O/e2e_${v}.json" 2>/dev/null
done
echo done > $O/done.txt
