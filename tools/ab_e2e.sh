#!/bin/bash
# e2e A/B of libcph.so builds on one box: bench.py (C4 x 21, 20 timed steps) per build, twice,
# printing ms/step, the device value and the e2e value.  usage: tools/ab_e2e.sh cur abtest/x.so ...
for k in 1 2; do
  for v in "$@"; do
    if [ "$v" == cur ]; then unset CPH_LIB; else export CPH_LIB=$v; fi
    python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
