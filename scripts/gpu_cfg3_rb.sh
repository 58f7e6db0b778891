OUT=gpurun_out/cfg3rb; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--config 3 --no-cpu-baseline --e2e-steps 0 --steps 200"
for rb in 32 64; do for tpg in 1 2 4 8; do
 timeout 120 python bench.py $B --tune run_bytes=$rb --tune tpg=$tpg > $OUT/rb${rb}_tpg$tpg.json 2>/dev/null
done; done
for tb in 32 64; do timeout 120 python bench.py $B --tune run_bytes=64 --tune thread_bytes=$tb > $OUT/rb64_tb$tb.json 2>/dev/null; done
