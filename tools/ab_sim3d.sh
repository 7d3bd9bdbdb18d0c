#!/bin/bash
# A/B of 3-D kernel variants selected by S3_FLAGS (bit 0: full Newton refactorization instead of the
# touched subtrees; bit 1: tree-level schedule (CSR tables); bit 2: tree-level schedule (register bit masks);
# bit 3: block barrier per substep; bit 4 / 5: block barrier before / after the Newton solve; bit 6: wave-
# balanced launch; defaults 40, plus 64 for models with nv >= 24 -- the G1 runs 104).
FLAGS=${FLAGS:-"104 105 72 64"}
for rep in 1 2; do
  for f in $FLAGS; do
    echo -n "flags=$f rep=$rep: "
    S3_FLAGS=$f timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --scale-envs 0 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('f32', j['sim3d']['f32']['ms_per_step'], 'f64', j['sim3d']['f64']['ms_per_step'])"
  done
done
