#!/usr/bin/env bash
# A/B of bench.py's device-timed draft level under environment variants: bash tools/ab_bench.sh "VAR=a" "VAR=b" ...
for v in "$@"; do
  for i in 1 2 3; do
    env $v timeout 300 python bench.py --no-cpu-baseline --no-decode 2>/dev/null | tail -1 | python -c "import sys,json; b=json.loads(sys.stdin.read()); print('$v', round(b['us_per_step'],2), round(b['e2e']['value']))"
  done
done
