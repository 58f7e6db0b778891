#!/bin/bash
# End-to-end: ramped chunk schedule (host_ramp) x chunk size x slots on
# config 5 against the PCIe ceiling; host-buffer parity tests.
O=gpurun_out/r02s3o
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "host" > $O/pytest.txt 2>&1
timeout 300 python scripts/pcie_probe.py > $O/pcie_probe.json 2> $O/pcie_probe.err
B="--no-cpu-baseline --also '' --ncu off --steps 50 --e2e-steps 8"
for v in "host_ramp=2" "host_ramp=0" "host_ramp=3" "host_ramp=0,host_chunk_mb=16" "host_ramp=2,host_chunk_mb=16" "host_ramp=3,host_chunk_mb=64" "host_ramp=2,host_chunk_mb=64"; do
  T=""; for kv in ${v//,/ }; do T="$T --tune $kv"; done
  for sm in 64 128; do
    eval timeout 300 python bench.py --config 5 $B $T --e2e-scratch-mb $sm > "$O/e2e_${v}_s${sm}.json" 2>/dev/null
  done
done
eval timeout 300 python bench.py --config 2 $B > "$O/e2e_cfg2.json" 2>/dev/null
echo done > $O/done.txt
