#!/bin/bash
# Round-2 final measurement bundle (GPU): the default bench line, the driver's
# 20-step line, ncu --set full of one round's kernels, the launch list.
set -x
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-cold > gpurun_out/bench20.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:sfg_mutate_kernel|sfg_jit_execute|sfg_jit_tail|sfg_stop_kernel|sfg_absorb_kernel|sfg_admit_kernel|sfg_dedupe|sfg_order_hist' \
    -s 60 -c 10 -o gpurun_out/prof_r02d python bench.py --steps 2 --warmup 6 --depth 1 --no-cpu --no-cold --no-sequential \
    > gpurun_out/ncu_r02d.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 800 -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --depth 8 --no-cpu --no-cold \
    --no-sequential > gpurun_out/ncu_launch.log 2>&1
true
