#!/bin/bash
# Config-3 access-pattern ceilings: the no-exchange variant of the compiled
# smem kernel under tile-shape knobs (run lengths, tile order, thread bytes),
# then the real conversion for the best shapes.
O=gpurun_out/r02s2o
mkdir -p $O
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for v in "" "run_bytes=512" "run_bytes=1024" "run_bytes_dst=128" "run_bytes_dst=256" "run_bytes=512,run_bytes_dst=128" \
         "run_bytes=512,run_bytes_dst=32" "run_bytes_dst=32" "tile_order=1" "tile_order=2" "auto_asym=0" \
         "thread_bytes=128" "thread_bytes=32" "run_bytes=1024,run_bytes_dst=64,thread_bytes=128"; do
  T=""; for kv in ${v//,/ }; do T="$T --tune $kv"; done
  eval timeout 300 python bench.py --config 3 $B $T --tune smem_jit_noxchg=1 > "$O/c3_noxchg_${v}.json" 2>/dev/null
  eval timeout 300 python bench.py --config 3 $B $T > "$O/c3_${v}.json" 2>/dev/null
done
echo done > $O/done.txt
