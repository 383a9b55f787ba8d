#!/bin/bash
# Round-end measurement bundle (GPU): default bench line, one ncu --set full
# capture of the bulk execute kernel, and the per-launch list of a short run.
set -x
[ -n "$SKIP_BENCH" ] || timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfg_jit_execute -s 3 -c 1 \
    -o gpurun_out/prof_bulk python bench.py --steps 1 --warmup 3 --depth 1 --no-cpu > gpurun_out/ncu_bulk.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:sfg_jit_tail -s 6 -c 1 \
    -o gpurun_out/prof_tail python bench.py --steps 1 --warmup 3 --depth 1 --no-cpu > gpurun_out/ncu_tail.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --depth 8 --no-cpu > gpurun_out/ncu_launch.log 2>&1
