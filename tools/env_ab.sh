#!/bin/bash
# Bench under several environment settings (GPU), REPS each, interleaved.
# Usage: CONFIGS="SFG_TAIL_K=1;SFG_TAIL_K=4" REPS=2 STEPS=20 bash tools/env_ab.sh
IFS=';' read -ra CF <<< "$CONFIGS"
for i in $(seq ${REPS:-2}); do
  for c in "${CF[@]}"; do
    v=$(env $c timeout 400 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu --no-cold --no-sequential --profile-rounds ${PROF:-2} 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k={x['kernel'][:8]: round(x['ms_per_round'],2) for x in (d.get('kernels') or [])}; print(round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2), k)")
    echo "[$c] rep $i: $v"
  done
done
