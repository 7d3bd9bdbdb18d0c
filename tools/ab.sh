#!/bin/bash
# A/B matrix of launch knobs: prints value, kernel_ms, e2e per setting.
# usage: tools/ab.sh "ENV=.. ENV2=.." "ENV=.." ...
for cfg in "$@"; do
  for rep in 1 2; do
    printf '%-50s ' "[$cfg]"
    env $cfg python bench.py --steps 300 --warmup 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1fM  kernel %.2f us  e2e %.1fM' % (d['value']/1e6, d['roofline']['kernel_ms']*1e3, d['e2e']['value']/1e6))"
  done
done
