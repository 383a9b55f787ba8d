#!/bin/bash
# Sweep the tail-pass configuration (inputs per warp, register cap) and the
# pipelining depth on the matmul workload.  GPU only.
for mb in ${MINBS:-16 24}; do
  for k in ${KS:-1 4}; do
    echo "== SFG_TAIL_MINB=$mb SFG_TAIL_K=$k"
    SFG_TAIL_MINB=$mb SFG_TAIL_K=$k CAPS= DEPTHS=${DEPTHS:-16,32,64} STEPS=${STEPS:-96} timeout 300 python tools/exec_probe.py matmul 65536
  done
done
