#!/bin/bash
# Round-2 measurement bundle (GPU): the default bench line; ncu --set full of one
# round's K1 / fused bulk / tail / triage kernels and of the seqgen kernels; the
# launch list of a short run; the L2 atomic peak probe.
set -x
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on \
    -k 'regex:sfg_mutate_kernel|sfg_plan_kernel|sfg_jit_execute|sfg_jit_tail|sfg_stop_kernel|sfg_absorb_kernel|sfg_admit_kernel' \
    -s 40 -c 9 -o gpurun_out/prof_r02b python bench.py --steps 2 --warmup 6 --depth 1 --no-cpu --no-cold --no-sequential \
    > gpurun_out/ncu_r02b.log 2>&1
timeout 600 ncu --set full --clock-control none -k 'regex:sfg_seq_walk|sfg_seq_mutate' -s 20 -c 2 \
    -o gpurun_out/prof_seq python tools/seq_probe.py matmul 4194304 1048576 > gpurun_out/ncu_seq.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 300 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --depth 8 --no-cpu --no-cold \
    --no-sequential > gpurun_out/ncu_launch.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_probe tools/atomic_probe.cu && /tmp/atomic_probe > gpurun_out/atomic_probe.txt 2>&1
true
