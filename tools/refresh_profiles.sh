#!/bin/bash
# Round profile refresh on the GPU box (round 2: the bench workload C4 x 21 replicas, default sub-batches):
# bench line, launch list of the same bench command, one ncu --set full capture of the step
# kernels at steady state (tools/prof_step.py, non-energy steps), CPH_TIMELINE stamps.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/prof/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra \
    > gpurun_out/prof/ncu_launch.log 2>&1
# per-kernel captures on whole-batch launches (one sub-batch: the kernels the S concurrent
# sub-batch launches add up to)
export CPH_CFG=4 CPH_R=21 CPH_STEPS=12 CPH_SUB_BATCHES=1
python tools/prof_step.py > gpurun_out/prof/plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_nonbonded|k_spread|k_gather|k_lambda_reduce|k_integrate|k_solve" \
    -s 12 -c 12 -o gpurun_out/prof/step_kernels python tools/prof_step.py > gpurun_out/prof/ncu_full.log 2>&1
# the rebuild kernels of the step-10 rebuild (the first matching launches are at create)
ncu --set full --clock-control none --import-source on -k regex:"k_build_list_col|k_cell_sort" \
    -s 2 -c 2 -o gpurun_out/prof/rebuild_kernels python tools/prof_step.py > gpurun_out/prof/ncu_rebuild.log 2>&1
unset CPH_SUB_BATCHES
CPH_TIMELINE=1 CPH_STEPS=100 python tools/prof_step.py > gpurun_out/prof/timeline.log 2>&1
ls -la gpurun_out/prof
