#!/bin/bash
# pair-list builder timing at C4 x 21 and C2 x 17 (bench per-class times), optional env variants
for k in 1 2; do
  for v in "${@:-CPH_X=0}"; do
    for cfg in "--config 4" "--config 2 --replicas 17"; do
      env $v python bench.py $cfg --steps 200 --warmup 20 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$v', '$cfg', round(d['ms_per_step'],4), 'rebuild', round(k['pairlist']['ms_per_rebuild'],4), 'nb', round(k['nonbonded']['ms_per_step'],4))"
    done
  done
done
