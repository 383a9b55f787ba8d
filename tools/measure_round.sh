#!/bin/bash
# Round measurement bundle (GPU, one call): bench line, long-input census, ncu launch
# list of a pipelined run, one ncu --set full capture per pipeline kernel.
# Usage: bash tools/measure_round.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
[ -n "$SKIP_BENCH" ] || timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
[ -n "$SKIP_LONG" ] || timeout 600 python tools/long_inputs.py matmul 262144 > gpurun_out/${tag}_long_inputs.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 8 --warmup 3 --depth 8 --no-cpu --no-cold \
    --profile-rounds 0 > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"sfg_jit_execute|sfg_jit_tail|sfg_mutate_kernel|sfg_apply_kernel|sfg_triage_absorb|sfg_plan_kernel" \
    -s 24 -c 8 -o gpurun_out/${tag}_kernels python bench.py --steps 2 --warmup 3 --depth 1 --no-cpu --no-cold \
    --profile-rounds 0 > gpurun_out/${tag}_ncu_full.log 2>&1
ls -la gpurun_out | tail -20
