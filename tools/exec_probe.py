"""Execute-kernel probe (GPU): K3 time per round for the scheduling modes and
block sizes, with the real budget and with a capped one (tail cost), plus the
retired-count distribution.  Usage: python tools/exec_probe.py [workload] [R]"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2603_05725_b200.lowering import VERDICT
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
m = load(name)
configs = [(mode, blk, bud) for mode in ("0", "1") for blk in ("128",) for bud in (1_000_000, 20_000)]
for mode, blk, bud in configs:
    os.environ["SFG_EXEC_MODE"], os.environ["SFG_EXEC_BLOCK"] = mode, blk
    from paper_2603_05725_b200.engine import DeviceCampaign
    dc = DeviceCampaign(m, master_seed=11, budget=bud)
    dc.timing = True
    it = 1
    dc.run_round(it, R); it += R
    k3 = []
    for _ in range(3):
        res = dc.run_round(it, R); it += R
        torch.cuda.synchronize()
        k3.append(res.slot.exec_ev[0].elapsed_time(res.slot.exec_ev[1]))
    v = res.slot.verdicts[:R * VERDICT.itemsize].cpu().numpy().view(VERDICT)
    ret = v["retired"].astype(np.int64)
    q = np.percentile(ret, [50, 90, 99, 99.9, 100]).astype(int).tolist()
    print(f"mode={mode} block={blk} budget={bud:>8d} k3_ms={[round(x, 2) for x in k3]} "
          f"execs/s={R / np.mean(k3) * 1e3:,.0f} retired p50/90/99/99.9/max={q} sum={ret.sum():,} "
          f"n_budget={(v['status'] == 2).sum()} sum_budget={ret[v['status'] == 2].sum():,}", flush=True)
    dc.close(); del dc; torch.cuda.empty_cache()
