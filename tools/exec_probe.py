"""Execute-kernel probe (GPU).  Part 1: K3 time per round (bulk + tail pass) vs
the deferral soft cap.  Part 2: pipelined step time vs rounds in flight.
Usage: python tools/exec_probe.py [workload] [R]"""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.lowering import VERDICT
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
m = load(name)
for cap in [int(x) for x in os.environ.get("CAPS", "0,8192,32768,131072").split(",") if x]:
    dc = DeviceCampaign(m, master_seed=11, soft_cap=cap)
    dc.timing = True
    it = 1
    dc.run_round(it, R); it += R
    k3 = []
    for _ in range(3):
        res = dc.run_round(it, R); it += R
        torch.cuda.synchronize()
        k3.append(res.slot.exec_ev[0].elapsed_time(res.slot.exec_ev[1]))
    nd = int(res.slot.counter[1].item()); nseq = int(res.slot.counter[3].item())
    bulk = res.slot.exec_ev[0].elapsed_time(res.slot.bulk_ev) if getattr(res.slot, "bulk_ev", None) else -1
    v = res.slot.verdicts[:R * VERDICT.itemsize].cpu().numpy().view(VERDICT)
    ret = v["retired"].astype(np.int64)
    print(f"soft_cap={cap:>7d} k3_ms={[round(x, 2) for x in k3]} execs/s={R / np.mean(k3) * 1e3:,.0f} "
          f"bulk_ms={bulk:.2f} deferred={nd} seq={nseq} retired_sum={ret.sum():,} max={ret.max():,}", flush=True)
    dc.close(); del dc; torch.cuda.empty_cache()

for depth in [int(x) for x in os.environ.get("DEPTHS", "8,16,32").split(",")]:
    dc = DeviceCampaign(m, master_seed=11)
    it = 1
    dc.run_rounds(it, it + 4 * R, R, depth=depth); it += 4 * R
    torch.cuda.synchronize()
    steps = int(os.environ.get("STEPS", "16"))
    t0 = time.perf_counter()
    res = dc.run_rounds(it, it + steps * R, R, depth=depth)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ex = sum(r.executed for r in res)
    print(f"depth={depth:3d} steps={steps} ms/step={dt / steps * 1e3:.2f} execs/s={ex / dt:,.0f} "
          f"mem_GB={torch.cuda.max_memory_allocated() / 1e9:.1f} admitted={sum(r.n_admitted for r in res)}",
          flush=True)
    dc.close(); del dc; torch.cuda.empty_cache()
