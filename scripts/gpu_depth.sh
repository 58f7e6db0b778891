#!/bin/bash
OUT=gpurun_out/depth; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/dp.py <<'PY'
import sys, random; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch, paper_2505_23819_b200 as ll
from test_gpu_parity import run_convert, expect_convert, rand_pair
from workloads import configs
ll.tune("smem_jit_depth", 2)
rng = random.Random(5)
cases = [configs.cfg2(batch_bits=3), configs.cfg3(n_bits=9), configs.cfg5(m_bits=9, kb_bits=9)] + [rand_pair(rng, rng.randint(12, 16), w) for w in (1, 2, 4, 8) for _ in range(3)]
ok = True
for c in cases:
    for batch in (1, 3):
        src, dst = run_convert(c, path="smem", batch=batch, seed=rng.randint(0, 99))
        ok &= dst.tobytes() == expect_convert(c, src, batch).tobytes()
print("depth2 parity", "OK" if ok else "FAIL")
PY
timeout 300 python /tmp/dp.py > $OUT/parity.txt 2>&1
B="--no-cpu-baseline --e2e-steps 0 --steps 300"
for c in 3 2 5; do for mb in 2 3; do
  timeout 200 python bench.py --config $c $B --tune smem_jit_depth=2 --tune smem_jit_minb=$mb > $OUT/cfg${c}_d2_minb$mb.json 2>/dev/null
done; timeout 200 python bench.py --config $c $B > $OUT/cfg${c}_d1.json 2>/dev/null; done
