#!/bin/bash
# Config-3 TMA plans with smaller tiles / fewer groups so that two
# destination images and 2-3 CTAs per SM fit (the persistent TMA-store
# kernel ran config 3 at 6380 GB/s-equivalent cold, alone, in ncu).
O=gpurun_out/r02s2k
mkdir -p $O
B="--no-cpu-baseline --e2e-steps 0 --also '' --ncu off --steps 300"
for p in smem_tma_store smem_tma; do
  for v in "tma_run_bytes_dst=128" "tma_run_bytes_dst=128,tmaj_k=1" "tma_run_bytes=128" "tma_run_bytes=128,tmaj_tpc=4" \
           "tmaj_tpc=-1,tmaj_cps=1" "tma_run_bytes_dst=128,tmaj_k=1,tmaj_tpc=4" "tma_run_bytes_dst=128,tmaj_tpc=-1,tmaj_cps=1,tmaj_stages=3" \
           "tma_run_bytes_dst=128,tmaj_k=1,tmaj_stages=3"; do
    T=""; for kv in ${v//,/ }; do T="$T --tune $kv"; done
    eval timeout 300 python bench.py --config 3 --path $p $B $T > "$O/c3_${p}_${v}.json" 2>/dev/null
  done
done
eval timeout 300 python bench.py --config 3 $B > $O/c3_auto.json 2>/dev/null
echo done > $O/done.txt
