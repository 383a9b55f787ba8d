"""e2e spread probe (GPU): fuzz_loop on the bench workload N times in one process
(after one bench-like device campaign), with the host clock of every round's
submission and finalization; prints each run's wall and, for slow runs, the
largest gaps.  Usage: SFG_ROUND_LOG=1 python tools/e2e_rounds.py [runs] [R]"""
import gc
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("SFG_ROUND_LOG", "1")
import torch  # noqa: E402
import paper_2603_05725_b200  # noqa: E402,F401
from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop  # noqa: E402
from paper_2603_05725_b200.workloads import load  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
m = load("matmul")
walls = []
for k in range(runs):
    torch.cuda.synchronize()
    gcn = gc.get_count()
    t0 = time.perf_counter()
    s = fuzz_loop(m, CampaignConfig(master_seed=11, iterations=48 * R, round_size=R, pipeline_depth=24))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    walls.append(wall)
    log = s.device_transfer.get("round_log", [])
    ev = [(n, r, t - t0) for n, r, t in log]
    gaps = sorted(((ev[i + 1][2] - ev[i][2], ev[i], ev[i + 1]) for i in range(len(ev) - 1)), reverse=True)[:6]
    print(f"run {k}: wall {wall:.3f} s, {s.compute_runs / wall / 1e6:.1f} M execs/s, gc {gcn}, "
          f"setup {s.device_transfer.get('setup_s', 0):.3f}, first event {ev[0][2] * 1e3:.1f} ms, "
          f"after last event {(wall - ev[-1][2]) * 1e3:.1f} ms" if ev else "")
    for g, a, b in gaps:
        print(f"    gap {g * 1e3:7.1f} ms  {a[0]} {a[1]} @ {a[2] * 1e3:.1f} -> {b[0]} {b[1]} @ {b[2] * 1e3:.1f}")
print("walls:", [round(w, 3) for w in walls])
