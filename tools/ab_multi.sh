#!/bin/bash
# same-box A/B of library builds: bash tools/ab_multi.sh lib1.so lib2.so ...  (base = in-tree)
for k in 1 2; do
  for lib in "" "$@"; do
    if [ -z "$lib" ]; then pre=""; name=base; else pre="CPH_LIB=$PWD/$lib"; name=$lib; fi
    env $pre python bench.py --steps 300 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$name', round(d['ms_per_step'],4), 'nb', round(k['nonbonded']['ms_per_launch'],4), 'list', round(k['pairlist']['ms_per_launch'],4))"
  done
done
