O=gpurun_out/e2echk; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for r in 1 2; do for k in 5 10 20; do
 timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps $k > $O/c3_k${k}_r$r.json 2>/dev/null
done; done
timeout 300 python bench.py --config 3 --no-cpu-baseline --e2e-steps 5 > $O/c3_default.json 2>/dev/null
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['e2e']['value'],1),round(d['e2e']['ms_per_step'],3))"; done > $O/summary.txt
