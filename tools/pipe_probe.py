"""Pipelined-round timeline without extra synchronization (GPU): per round, when
its execute pass started, when the bulk pass and the tail passes ended (CUDA
events on the round's stream, read after the run), plus deferral counts.
Usage: python tools/pipe_probe.py [workload] [R] [depth] [steps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 32
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 64
dc = DeviceCampaign(load(name), master_seed=11)
dc.run_rounds(1, 1 + 4 * R, R, depth=depth)
torch.cuda.synchronize()
dc.timing = True
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
rows = []
host0 = time.perf_counter()


slowest = []


def on_round(res):
    S = res.slot
    from paper_2603_05725_b200.lowering import VERDICT
    nd = int(S.counter[1].item())
    if nd:
        d = S.deferred[:nd].cpu().numpy()
        v = S.verdicts[:S.n * VERDICT.itemsize].cpu().numpy().view(VERDICT)
        ns = (v["where"][d] >> 9).astype(np.int64)
        j = int(np.argmax(ns))
        i = int(d[j])
        slowest.append((float(ns[j]) / 1e6, int(v["retired"][i]), int((v["where"][i] >> 8) & 1), int(v["status"][i]),
                        len(slowest), dc.child_testcases([i], S)[0]))
    rows.append((S.exec_ev, getattr(S, "bulk_ev", None), S.counter[:8].clone(), time.perf_counter() - host0,
                 S.sub_ev, S.sub_host - host0))


it = 1 + 4 * R
res = dc.run_rounds(it, it + steps * R, R, depth=depth, on_round=on_round)
torch.cuda.synchronize()
wall = time.perf_counter() - host0
out = []
for (s, e), b, cnt, h, sub, subh in rows:
    c = cnt.cpu().numpy()
    out.append((t0.elapsed_time(s), t0.elapsed_time(b) if b else -1, t0.elapsed_time(e), h * 1e3, c[1], c[3],
                t0.elapsed_time(sub), subh * 1e3))
a = np.array(out)
print(f"{name} R={R} depth={depth} steps={steps}: wall/step={wall / steps * 1e3:.2f} ms "
      f"execs/s={sum(r.executed for r in res) / wall:,.0f}")
print(f"  bulk dur ms: mean {np.mean(a[:, 1] - a[:, 0]):.2f} max {np.max(a[:, 1] - a[:, 0]):.2f}; "
      f"tail dur ms: mean {np.mean(a[:, 2] - a[:, 1]):.2f} max {np.max(a[:, 2] - a[:, 1]):.2f}; "
      f"deferred mean {a[:, 4].mean():.0f} seq mean {a[:, 5].mean():.0f}")
slowest.sort(key=lambda x: -x[0])
print("slowest long input per round (ms, retired, rerun, status, round, scalar args):")
for ms, ret, rr, st, k, tc in slowest[:12]:
    print(f"  {ms:7.1f} {ret:>10,} {rr} {st} r{k} {[a.value if hasattr(a, 'value') else len(a.data) for a in tc.args]}")
print("round  host_submit  gpu_submit  exec_start  bulk_end  tail_end  host_final  n_def  n_seq")
for k, r in enumerate(out):
    print(f"{k:5d} {r[7]:12.1f} {r[6]:11.1f} {r[0]:11.1f} {r[1]:9.1f} {r[2]:9.1f} {r[3]:11.1f} {int(r[4]):6d} {int(r[5]):6d}")
