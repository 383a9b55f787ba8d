#!/bin/bash
# bench at several round-in-flight depths (GPU): device-timed and end-to-end M execs/s
for d in ${DEPTHS:-24 12 8}; do
  for r in $(seq ${REPS:-2}); do
    v=$(timeout 300 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu --no-cold --no-sequential --depth $d 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1))")
    echo "depth $d rep $r: $v"
  done
done
