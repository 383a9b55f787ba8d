#!/bin/bash
# Device-timed / e2e spread of the default bench (GPU): REPS runs per setting, with
# the per-round host timeline of each run kept (gpurun_out/var_<tag>_<i>.tl).
IFS=';' read -ra CF <<< "${CONFIGS:-X=1;SFG_BENCH_NO_NVML=1}"
for i in $(seq ${REPS:-4}); do
  for c in "${CF[@]}"; do
    tag=$(echo "$c" | tr -c 'A-Za-z0-9' '_')
    v=$(env $c SFG_BENCH_TIMELINE=gpurun_out/var_${tag}_$i.tl timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu --no-cold --no-sequential --profile-rounds 0 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2), round(d['e2e']['wall_s'],3))")
    echo "[$c] rep $i: $v"
  done
done
