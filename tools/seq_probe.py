"""Sequential-discipline throughput probe (GPU): fuzz_loop(discipline="sequential")
on a workload at several round sizes; prints execs/s, rounds, seqgen truncations."""
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import torch  # noqa: E402
from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop  # noqa: E402
from paper_2603_05725_b200.workloads import load  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
execs = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
sizes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1 << 16, 1 << 18, 1 << 20]
m = load(name)
fuzz_loop(m, CampaignConfig(master_seed=11, iterations=1 << 14, discipline="sequential", round_size=1 << 12))
for R in [r for r in sizes for _ in range(2)]:   # each size twice: the second with warm buffers
    torch.cuda.synchronize()
    t = time.perf_counter()
    s = fuzz_loop(m, CampaignConfig(master_seed=11, iterations=execs, discipline="sequential", round_size=R))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    dtf = s.device_transfer
    print(f"{name} R={R}: {s.compute_runs / dt / 1e6:.2f} M execs/s ({s.compute_runs} in {dt:.2f} s, rounds {dtf['rounds']}, "
          f"corpus {s.corpus.interesting}, findings {len(s.findings)})", flush=True)
