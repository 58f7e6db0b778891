#!/bin/bash
# A/B: compiled smem kernel with one staging buffer per group (smem_jit_single,
# half the shared memory; launches with one tile per group) x register cap.
set -u
OUT=gpurun_out/single
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
cat > /tmp/sp.py <<'PY'
import sys, random; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2505_23819_b200 as ll
from test_gpu_parity import run_convert, expect_convert, rand_pair
from workloads import configs
ll.tune("smem_jit_single", 1)
rng = random.Random(7)
cases = [configs.cfg2(batch_bits=3), configs.cfg3(n_bits=9), configs.cfg5(m_bits=9, kb_bits=9)] + [rand_pair(rng, rng.randint(12, 16), w) for w in (1, 2, 4, 8) for _ in range(3)]
ok = True
for c in cases:
    for batch in (1, 3):
        src, dst = run_convert(c, path="smem", batch=batch, seed=rng.randint(0, 99))
        ok &= dst.tobytes() == expect_convert(c, src, batch).tobytes()
print("single parity", "OK" if ok else "FAIL")
PY
timeout 300 python /tmp/sp.py > $OUT/parity.txt 2>&1
for rep in 1 2; do
  for c in 3 2 5; do
    for v in "def:" "s1:--tune smem_jit_single=1" "s1m4:--tune smem_jit_single=1 --tune smem_jit_minb=4" \
             "s1m5:--tune smem_jit_single=1 --tune smem_jit_minb=5" "s1m3:--tune smem_jit_single=1 --tune smem_jit_minb=3"; do
      n=${v%%:*}; a=${v#*:}
      timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 $a \
        > $OUT/cfg${c}_${n}_r$rep.json 2> $OUT/cfg${c}_${n}_r$rep.err
    done
  done
done
python - <<'PY'
import json, glob, os
rows = {}
for f in sorted(glob.glob("gpurun_out/single/cfg*_r*.json")):
    k = os.path.basename(f).rsplit("_r", 1)[0]
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        rows.setdefault(k, []).append((round(d["value"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
    except Exception as e:
        rows.setdefault(k, []).append(str(e)[:60])
for k, v in sorted(rows.items()): print(k, v)
json.dump(rows, open("gpurun_out/single/summary.json", "w"), indent=1)
PY
