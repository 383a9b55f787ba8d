"""Pipelined-round timeline (GPU): per round, when its bulk pass and tail pass
ended relative to the first submission; where (SM) and how long the deferred
inputs ran.  Usage: python tools/timeline.py [depth] [R] [soft_cap]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import collections
import numpy as np
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.lowering import VERDICT
from paper_2603_05725_b200.workloads import load

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 16
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
dc = DeviceCampaign(load("matmul"), master_seed=11, soft_cap=cap)
dc.run_rounds(1, 1 + 2 * R, R, depth=depth)
torch.cuda.synchronize()
dc.timing = True
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
rows = []
host0 = time.perf_counter()


def on_round(res):
    S = res.slot
    torch.cuda.synchronize()
    s, e = S.exec_ev
    b = getattr(S, "bulk_ev", None)
    nd = int(S.counter[1].item())
    v = S.verdicts[:S.n * VERDICT.itemsize].cpu().numpy().view(VERDICT)
    d = S.deferred[:nd].cpu().numpy()
    w = v["where"][d] if nd else np.zeros(0, np.uint64)
    sms = collections.Counter((w & 0xff).tolist())
    dur = (w >> 9) / 1e6
    rows.append((t0.elapsed_time(s), t0.elapsed_time(b) if b else -1, t0.elapsed_time(e),
                 (time.perf_counter() - host0) * 1e3, nd, len(sms), max(sms.values()) if sms else 0,
                 float(dur.max()) if nd else 0, float(np.median(dur)) if nd else 0,
                 float(((v["where"] >> 9) / 1e6).max())))


it = 1 + 2 * R
steps = 3 * depth
t_start = time.perf_counter()
dc.run_rounds(it, it + steps * R, R, depth=depth, on_round=on_round)
torch.cuda.synchronize()
print(f"depth={depth} R={R} soft_cap={cap} wall/step={(time.perf_counter() - t_start) / steps * 1e3:.1f} ms "
      "(includes per-round sync in this probe)")
print("round  start  bulk_end  tail_end  host_fin  n_def  tail_SMs  max/SM  tail_max_ms  tail_med_ms  input_max_ms")
for k, r in enumerate(rows):
    print(f"{k:5d} {r[0]:7.1f} {r[1]:9.1f} {r[2]:9.1f} {r[3]:9.1f} {r[4]:6d} {r[5]:9d} {r[6]:7d} {r[7]:11.1f} {r[8]:11.1f} {r[9]:11.1f}")
