python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
mkdir -p gpurun_out/gv8
LL_GATHER_V8=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gather" > gpurun_out/gv8/pytest.txt 2>&1
B="--config 4 --no-cpu-baseline --e2e-steps 0 --steps 500"
for r in 1 2; do
  timeout 200 python bench.py $B > gpurun_out/gv8/v4_$r.json 2>/dev/null
  for vpt in 1 2; do timeout 200 python bench.py $B --tune gather_v8=1 --tune gather_vpt=$vpt > gpurun_out/gv8/v8_vpt${vpt}_$r.json 2>/dev/null; done
done
