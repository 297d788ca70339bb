#!/bin/bash
mkdir -p gpurun_out
for k in 1 2 3; do
  for v in "CPH_X=0" "CPH_PRIO_SWAP=1" "CPH_NO_PRIO=1"; do
    env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$v', round(d['ms_per_step'],4), 'nb', round(k['nonbonded']['ms_per_launch'],4), d['clocks']['sm_mhz'])"
  done
done
for v in "CPH_X=0" "CPH_PRIO_SWAP=1"; do
  echo "== timeline $v"
  env $v CPH_TIMELINE=1 python bench.py --steps 200 --warmup 20 --no-cpu-baseline 2>&1 >/dev/null | grep timeline | tail -10
done
