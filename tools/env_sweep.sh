#!/bin/bash
# Bench under several environment settings (GPU): CONFIGS="name:VAR=v,VAR=v ..."
R=$GRAFT_REPO_ROOT
for rep in $(seq ${REPS:-2}); do
  for c in $CONFIGS; do
    name=${c%%:*}; envs=${c#*:}; envs=${envs//,/ }
    (cd $R && env $envs timeout 300 python bench.py --no-cpu > gpurun_out/sweep_${name}_$rep.log 2>&1)
  done
done
