#!/bin/bash
# Config-3 run-length sweep: reversed asymmetry (short source runs, long
# destination runs) and symmetric 128-byte runs, with both tile orders.
O=gpurun_out/r02s3d
mkdir -p $O
S=";run_bytes_src=64,run_bytes_dst=256;run_bytes_src=64,run_bytes_dst=256,tile_order=1;run_bytes_src=128,run_bytes_dst=128"
S="$S;run_bytes_src=128,run_bytes_dst=128,tile_order=1;run_bytes_src=128,run_bytes_dst=256;run_bytes_src=128,run_bytes_dst=256,tile_order=1"
S="$S;run_bytes_src=32,run_bytes_dst=256;run_bytes=512,run_bytes_src=64,run_bytes_dst=512;tile_order=12"
timeout 1200 python scripts/ab_knobs.py 3 "$S" 5 >> $O/ab_runs.jsonl 2>> $O/ab_runs.err
echo done > $O/done.txt
