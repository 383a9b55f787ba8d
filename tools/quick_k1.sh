#!/bin/bash
# K1 A/B on the GPU box: bench stage timings + one ncu capture of plan/mutate.
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-cold --no-sequential > gpurun_out/qb.log 2> gpurun_out/qb.err
timeout 600 ncu --set full --clock-control none -k 'regex:sfg_mutate_kernel|sfg_plan_kernel' -s 4 -c 2 \
    -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 4 --depth 1 --no-cpu --no-cold --no-sequential \
    > gpurun_out/ncu_k1.log 2>&1
true
