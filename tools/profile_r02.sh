#!/bin/bash
# One ncu --set full capture of a round's streaming kernels and bulk pass
# (K1 sfg_mutate, K2 sfg_apply, K3 bulk sfg_jit_execute, the tail's re-materialize),
# source-correlated; plus the launch list of a short run.
set -x
timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:sfg_mutate_kernel|sfg_apply_kernel|sfg_jit_execute|sfg_plan_kernel' -s 15 -c 5 \
    -o gpurun_out/prof_r02 python bench.py --steps 2 --warmup 4 --depth 1 --no-cpu --no-cold --no-sequential \
    > gpurun_out/ncu_r02.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 300 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --depth 8 --no-cpu --no-cold \
    --no-sequential > gpurun_out/ncu_launch.log 2>&1
