run() { echo "== $E $*"; env $E timeout 400 python bench.py --no-cpu "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3gM e2e %.3gM k3 %.1f max %.1f bulk %.2f' % (d['value']/1e6, d['e2e']['value']/1e6, d['issue_roofline']['k3_ms_per_round'], d['issue_roofline']['k3_ms_per_round_max'], d['roofline']['launch_ms']))"; }
E="SFG_TAIL_MINB=12" run
E="SFG_TAIL_MINB=16" run
E="SFG_TAIL_MINB=20" run
E="SFG_TAIL_MINB=16" run
E="SFG_TAIL_MINB=12" run
