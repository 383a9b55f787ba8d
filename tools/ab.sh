run() { echo "== $E $*"; env $E timeout 400 python bench.py --no-cpu "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3gM e2e %.3gM k3 %.1f max %.1f bulk %.2f' % (d['value']/1e6, d['e2e']['value']/1e6, d['issue_roofline']['k3_ms_per_round'], d['issue_roofline']['k3_ms_per_round_max'], d['roofline']['launch_ms']))"; }
E="X=1" run
E="X=1" run
E="X=1" run
timeout 600 ncu --set full --clock-control none -k regex:sfg_jit_execute -s 3 -c 1 -o gpurun_out/prof_bulk_mag python bench.py --steps 1 --warmup 3 --depth 1 --no-cpu > /dev/null 2>&1
