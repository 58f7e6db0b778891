#!/bin/bash
# Session-3 defaults (PDL prefetch, shuffle PDL, gather PDL): classification
# rows, interleaved A/B of every path on every config, default line.
O=gpurun_out/r02s3i
mkdir -p $O
timeout 900 python scripts/classify_bench.py > $O/classify.json 2> $O/classify_rows.jsonl
timeout 1200 python scripts/ab_paths.py 3 > $O/ab_paths.jsonl 2> $O/ab_paths.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo done > $O/done.txt
