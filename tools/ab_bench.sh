#!/bin/bash
# A/B of two configurations of the bench (GPU): $A_ENV / $B_ENV are environment
# assignments, or B_DIR a second checkout (built) to compare against this one.
# Each run also writes its per-round timeline (gpurun_out/ab_{a,b}_<i>.tl).
set -x
R=$GRAFT_REPO_ROOT
for i in $(seq ${REPS:-2}); do
  (cd $R && env $A_ENV SFG_BENCH_TIMELINE=$R/gpurun_out/ab_a_$i.tl timeout 300 python bench.py --no-cpu > gpurun_out/ab_a_$i.log 2>&1)
  (cd $R/${B_DIR:-.} && env $B_ENV SFG_BENCH_TIMELINE=$R/gpurun_out/ab_b_$i.tl timeout 300 python bench.py --no-cpu > $R/gpurun_out/ab_b_$i.log 2>&1)
done
