#!/bin/bash
O=gpurun_out/r02s3m
mkdir -p $O
timeout 300 python scripts/pcie_probe.py > $O/pcie_probe.json 2> $O/pcie_probe.err
echo done > $O/done.txt
