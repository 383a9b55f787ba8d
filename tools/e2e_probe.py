"""End-to-end variance probe (GPU): fuzz_loop repeated in one process, and the
same campaign through DeviceCampaign.run_rounds, wall-clocked.
Usage: python tools/e2e_probe.py [R] [depth] [rounds]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_05725_b200  # noqa: F401
import torch
from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.workloads import load

R = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
D = int(sys.argv[2]) if len(sys.argv) > 2 else 24
K = int(sys.argv[3]) if len(sys.argv) > 3 else 32
m = load("matmul")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dc = DeviceCampaign(m, master_seed=11)
    t1 = time.perf_counter()
    res = dc.run_rounds(1, 1 + K * R, R, depth=D)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dc.close()
    print(f"run_rounds rep{rep}: create {t1 - t0:.3f}s rounds {t2 - t1:.3f}s -> {K * R / (t2 - t0) / 1e6:.2f}M/s", flush=True)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = fuzz_loop(m, CampaignConfig(master_seed=11, iterations=K * R, round_size=R, pipeline_depth=D))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"fuzz_loop rep{rep}: {dt:.3f}s -> {s.compute_runs / dt / 1e6:.2f}M/s", flush=True)
