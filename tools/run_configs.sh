#!/bin/bash
# every BASELINE config at its batched operating points (300 timed steps, no CPU baseline)
mkdir -p gpurun_out/configs
for cr in "1 64" "1 256" "2 17" "2 68" "3 45" "4 21" "5 1" "5 8"; do
  set -- $cr
  timeout 600 python bench.py --config $1 --replicas $2 --steps 300 --warmup 20 --no-cpu-baseline --no-extra --e2e-steps 2 \
      > gpurun_out/configs/cfg_$1_$2.json 2> gpurun_out/configs/cfg_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/configs/cfg_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],4), round(d['ns_per_day_per_system'],1), round(d['value'],1))"
done
