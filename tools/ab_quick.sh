#!/bin/bash
# quick same-box timing of the two headline workloads (bench per-class times)
for k in 1 2 3; do
  for cfg in "--config 4" "--config 2 --replicas 17"; do
    python bench.py $cfg --steps 200 --warmup 20 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$cfg', round(d['ms_per_step'],4), 'nb', round(k['nonbonded']['ms_per_step'],4), 'rebuild', round(k['pairlist']['ms_per_rebuild'],4))"
  done
done
