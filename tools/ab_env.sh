#!/bin/bash
# same-box A/B of environment switches: bash tools/ab_env.sh "CPH_X=0" "CPH_FOO=1" ...
for k in 1 2 3; do
  for v in "$@"; do
    env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['ms_per_step'],4), 'nb', round(k['nonbonded']['ms_per_launch'],4), 'lam', round(k['lambda']['ms_per_launch'],4), d['clocks']['sm_mhz'])"
  done
done
for v in "$@"; do
  echo "== timeline $v"
  env $v CPH_TIMELINE=1 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 >/dev/null | grep timeline | tail -3
done
