"""Which host call blocks round submission (GPU)?  Runs the bench's pipelined
campaign (matmul, rounds of 262,144, 24 in flight) with every sfg_* C-ABI call
timed on the host; prints the calls that took longer than 5 ms.
Usage: python tools/submit_probe.py [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_05725_b200  # noqa: F401
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.workloads import load

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
R, D, K = 262144, 24, 96
dc = DeviceCampaign(load("matmul"), master_seed=11)
slow = []
t_origin = [0.0]
for name in [n for n in dir(dc.L) if n.startswith("sfg_")] + ["sfg_execute", "sfg_execute_deferred", "sfg_mutate",
                                                              "sfg_plan", "sfg_apply", "sfg_order", "sfg_scan_u32",
                                                              "sfg_scan_u64", "sfg_triage_stop", "sfg_triage_absorb",
                                                              "sfg_triage_admit", "sfg_commit"]:
    f = getattr(dc.L, name)
    if not callable(f) or getattr(f, "_wrapped", False):
        continue

    def wrap(f=f, name=name):
        def g(*a):
            t = time.perf_counter()
            r = f(*a)
            dt = time.perf_counter() - t
            if dt > 0.005:
                slow.append((name, round((t - t_origin[0]) * 1e3, 1), round(dt * 1e3, 1)))
            return r
        g._wrapped = True
        return g
    setattr(dc.L, name, wrap())
it = 1
dc.run_rounds(it, it + 3 * R, R, depth=D)
it += 3 * R
for rep in range(reps):
    dc.reserve(D, R)
    torch.cuda.synchronize()
    slow.clear()
    t_origin[0] = time.perf_counter()
    dc.run_rounds(it, it + K * R, R, depth=D)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t_origin[0]
    it += K * R
    print(f"rep{rep}: {K * R / dt / 1e6:.1f}M/s wall {dt * 1e3:.0f} ms; slow calls (name, start ms, ms): {slow[:30]}",
          flush=True)
