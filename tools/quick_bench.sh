#!/bin/bash
# Quick A/B on the GPU box: the default bench line without the CPU / cold / sequential
# legs, then one ncu --set full capture of the bulk pass and K1 (source-correlated).
set -x
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-cold --no-sequential > gpurun_out/qb.log 2> gpurun_out/qb.err
[ -n "$NO_NCU" ] || timeout 600 ncu --set full --clock-control none --import-source on \
    -k 'regex:sfg_mutate_kernel|sfg_jit_execute|sfg_plan_kernel|sfg_apply_kernel' -s 12 -c 4 \
    -o gpurun_out/prof_q python bench.py --steps 2 --warmup 4 --depth 1 --no-cpu --no-cold --no-sequential \
    > gpurun_out/ncu_q.log 2>&1
true
