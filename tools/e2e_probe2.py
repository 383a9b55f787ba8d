"""Run-to-run variance probe (GPU): the same campaign repeated on one
DeviceCampaign, then on fresh ones.  Usage: python tools/e2e_probe2.py [R] [depth] [rounds]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_05725_b200  # noqa: F401
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.workloads import load

R = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
D = int(sys.argv[2]) if len(sys.argv) > 2 else 24
K = int(sys.argv[3]) if len(sys.argv) > 3 else 48
m = load("matmul")
dc = DeviceCampaign(m, master_seed=11)
it = 1
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dc.run_rounds(it, it + K * R, R, depth=D)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it += K * R
    print(f"same dc rep{rep}: {dt:.3f}s -> {K * R / dt / 1e6:.2f}M/s admitted={sum(r.n_admitted for r in res)}", flush=True)
dc.close()
for rep in range(4):
    dc = DeviceCampaign(m, master_seed=11)
    dc.reserve(D, R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dc.run_rounds(1, 1 + K * R, R, depth=D)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"fresh dc rep{rep}: {dt:.3f}s -> {K * R / dt / 1e6:.2f}M/s admitted={sum(r.n_admitted for r in res)}", flush=True)
    dc.close()
    del dc
