#!/bin/bash
# Round profile refresh on the GPU box: bench line, launch list of the same command, one
# ncu --set full capture per step kernel (C2 x 17 replicas via tools/prof_step.py).
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err || exit 1
python bench.py --steps 2 --warmup 3 > gpurun_out/prof/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/prof/ncu_launch.log 2>&1
CPH_STEPS=12 python tools/prof_step.py > gpurun_out/prof/plain_step.log 2>&1 || exit 1
for k in k_nonbonded k_build_list k_spread k_gather k_lambda_reduce k_integrate k_solve k_cell_sort; do
  CPH_STEPS=12 ncu --set full --clock-control none --import-source on -k regex:"$k\b" -s 1 -c 1 \
      -o gpurun_out/prof/$k python tools/prof_step.py > gpurun_out/prof/ncu_$k.log 2>&1
done
ls -la gpurun_out/prof
