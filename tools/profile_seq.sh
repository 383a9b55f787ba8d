#!/bin/bash
# Sequential discipline on the GPU box: throughput probe + launch list of the seqgen kernels.
timeout 600 python tools/seq_probe.py matmul 33554432 262144,1048576 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sfg_seq|sfg_jit|sfg_apply|sfg_mutate' -s 300 -c 200 --csv \
    --log-file gpurun_out/seq_launches.csv python tools/seq_probe.py matmul 8388608 1048576 > gpurun_out/seq_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/seq_launches.csv 2>&1 | head -16
