#!/bin/bash
# in-situ bank conflicts without global loads AND stores; cfg3 launch / plan sweep
O=gpurun_out/r02f
mkdir -p $O
B="--no-cpu-baseline --e2e-steps 0 --also '' --steps 300"
for c in 2 3 5; do
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_noload=1 --tune smem_jit_nostore=1 --ncu on > $O/bench_cfg${c}_nols.json 2> $O/bench_cfg${c}_nols.err
  eval timeout 300 python bench.py --config $c $B --tune smem_jit_nostore=1 --ncu on > $O/bench_cfg${c}_nost.json 2> $O/bench_cfg${c}_nost.err
done
B="$B --ncu off"
for t in "tile_order=1" "tile_order=2" "run_bytes_dst=128" "run_bytes_dst=256" "thread_bytes=128" "smem_jit_depth=2" "smem_jit_tpg=2" "smem_jit_minb=2" "pdl=0" "auto_asym=0" "run_bytes=512"; do
  eval timeout 300 python bench.py --config 3 $B --tune $t > $O/sweep3_$t.json 2>/dev/null
done
echo done > $O/done.txt
