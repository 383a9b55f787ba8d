#!/bin/bash
# Group-parallel vs thread-sequential execute on one workload (GPU).
W=${1:-matmul}
for g in ${GROUPS_:-1 8}; do
  echo "== SFG_GROUP=$g"
  SFG_GROUP=$g CAPS=${CAPS:-32768} DEPTHS=${DEPTHS:-32} STEPS=${STEPS:-64} timeout 300 python tools/exec_probe.py $W 65536
done
