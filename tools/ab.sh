run() { echo "== $E $*"; env $E timeout 400 python bench.py --no-cpu "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3gM e2e %.3gM k3 %.1f max %.1f bulk %.2f' % (d['value']/1e6, d['e2e']['value']/1e6, d['issue_roofline']['k3_ms_per_round'], d['issue_roofline']['k3_ms_per_round_max'], d['roofline']['launch_ms']))"; }
E="SFG_TAIL_K=4" run
E="SFG_TAIL_K=4 SFG_TAIL_CTAS=512" run
E="SFG_GROUP=4 SFG_TAIL_K=8" run
E="SFG_GROUP=2 SFG_TAIL_K=16" run
E="SFG_GROUP=1 SFG_TAIL_K=32" run
E="SFG_TAIL_K=4" run --depth 28
