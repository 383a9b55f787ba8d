"""Host-side profile of the pipelined round loop (GPU): where the Python host
spends its time per round (cProfile, top functions by own time).
Usage: python tools/host_profile.py [workload] [R] [depth] [steps]"""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 32
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 96
dc = DeviceCampaign(load(name), master_seed=11)
dc.run_rounds(1, 1 + 4 * R, R, depth=depth)
torch.cuda.synchronize()
it = 1 + 4 * R
pr = cProfile.Profile()
t0 = time.perf_counter()
c0 = time.process_time()
pr.enable()
res = dc.run_rounds(it, it + steps * R, R, depth=depth)
torch.cuda.synchronize()
pr.disable()
dt = time.perf_counter() - t0
print(f"wall/step={dt / steps * 1e3:.2f} ms  cpu/step={(time.process_time() - c0) / steps * 1e3:.2f} ms  "
      f"execs/s={sum(r.executed for r in res) / dt:,.0f} (profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
