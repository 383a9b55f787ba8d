"""Execute-kernel time vs round size, and the retired-count distribution (GPU)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.lowering import VERDICT
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
m = load(name)
for R in [int(x) for x in (sys.argv[2:] or ["4096", "16384", "65536", "262144", "1048576"])]:
    dc = DeviceCampaign(m, master_seed=11)
    dc.timing = True
    it = 1
    dc.run_round(it, R); it += R   # warm
    times = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); res = dc.run_round(it, R); e.record(); torch.cuda.synchronize()
        it += R
        times.append((s.elapsed_time(e), res.slot.exec_ev[0].elapsed_time(res.slot.exec_ev[1])))
    v = res.slot.verdicts[:R * VERDICT.itemsize].cpu().numpy().view(VERDICT)
    ret = v["retired"].astype(np.int64)
    q = np.percentile(ret, [50, 90, 99, 99.9, 100])
    print(f"R={R:8d} step_ms={[round(t[0],2) for t in times]} k3_ms={[round(t[1],2) for t in times]} "
          f"execs/s={R/np.mean([t[0] for t in times])*1e3:,.0f} retired p50/90/99/99.9/max={q.astype(int).tolist()} "
          f"sum={ret.sum():,} budget={(v['status']==2).sum()}", flush=True)
    dc.close()
    del dc
    torch.cuda.empty_cache()
