#!/bin/bash
# A/B of 3-D kernel variants selected by S3_FLAGS, alternating, same box.
for rep in 1 2; do
  for f in 0 1; do  # 0: partial refactorization, 1: full
    echo -n "flags=$f rep=$rep: "
    S3_FLAGS=$f timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --scale-envs 0 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['sim3d']['f32']['ms_per_step'], j['sim3d']['f64']['ms_per_step'])"
  done
done
