#!/bin/bash
# K1 (sfg_mutate_kernel) launch times of several built checkouts under abtest/ (GPU).
R=$GRAFT_REPO_ROOT
for v in ${VARIANTS:-a b c}; do
  (cd $R/abtest/$v && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sfg_mutate_kernel \
     -s 3 -c 6 --csv python bench.py --steps 3 --warmup 3 --depth 1 --no-cpu > $R/gpurun_out/k1_$v.csv 2>&1)
done
