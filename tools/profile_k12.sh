#!/bin/bash
# ncu --set full of the streaming kernels (K1 mutate, K2 apply) in the 4th round.
for k in sfg_mutate_kernel sfg_apply_kernel sfg_plan_kernel; do
timeout 300 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 3 --depth 1 --no-cpu > gpurun_out/ncu_$k.log 2>&1
done
