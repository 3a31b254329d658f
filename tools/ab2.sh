#!/usr/bin/env bash
# A/B of the C2 draft level under environment variants (3 runs each):
#   bash tools/ab2.sh "VAR=a" "VAR=b" ...   -> steady us/step, isolated p50, e2e steps/s
for v in "$@"; do
  for i in 1 2 3; do
    env $v timeout 300 python bench.py --no-cpu-baseline --no-decode --no-verify --no-sweep --no-batched --steps 1000 2>/dev/null | tail -1 | python -c "
import sys,json; b=json.loads(sys.stdin.read()); r=b['roofline']
print('$v', round(b['us_per_step'],2), round(r['chain_us_isolated_pct']['p50'],2), round(b['e2e']['value']), round(r['frac'],3))"
  done
done
