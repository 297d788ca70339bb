#!/bin/bash
# A/B timing: alternate runs of bench.py with and without an environment switch
for k in 1 2 3; do
  for v in "" "$1"; do
    env $v python bench.py --steps 300 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${v:-base}', round(d['ms_per_step'],4), round(d['kernels']['nonbonded']['ms_per_launch'],4))"
  done
done
