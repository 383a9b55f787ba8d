"""fuzz_loop end-to-end variance (GPU): repeated campaigns with a per-round
finalize timeline of the slowest one.  Usage: python tools/e2e_probe3.py [R] [depth] [rounds] [reps]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_05725_b200  # noqa: F401
import torch
from paper_2603_05725_b200 import engine
from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
from paper_2603_05725_b200.workloads import load

R = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
D = int(sys.argv[2]) if len(sys.argv) > 2 else 24
K = int(sys.argv[3]) if len(sys.argv) > 3 else 192
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
m = load("matmul")
orig = engine.DeviceCampaign._finalize
log = []


def fin(self, S):
    res = orig(self, S)
    log.append((time.perf_counter(), res.n_admitted, self.spec_depth))
    return res


engine.DeviceCampaign._finalize = fin
if "--after-bench" in sys.argv:
    # the bench's order: a device-timed campaign first, its buffers released
    import gc
    dc = engine.DeviceCampaign(m, master_seed=11)
    dc.run_rounds(1, 1 + 99 * R, R, depth=D)
    dc.close(); dc.slots.clear(); dc._aux = None
    del dc
    gc.collect()
gc_off = "--gc-off" in sys.argv
runs = []
for rep in range(reps):
    log.clear()
    torch.cuda.synchronize()
    a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    import gc
    if gc_off:
        gc.disable()
    t0 = time.perf_counter()
    s = fuzz_loop(m, CampaignConfig(master_seed=11, iterations=K * R, round_size=R, pipeline_depth=D))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    gc.enable()
    gaps = [b[0] - a[0] for a, b in zip(log, log[1:])]
    adm = [k for k, x in enumerate(log) if x[1]]
    runs.append((dt, list(log), t0))
    rl = s.device_transfer.get("round_log")
    if rl:
        marks = {n: t for n, k, t in rl if k == -1}
        tail = {n: round((t - t0) * 1e3) for n, t in marks.items()}
        print("   phases (ms from call):", tail, "last finalize", round((log[-1][0] - t0) * 1e3),
              "end", round(dt * 1e3))
    a1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    print(f"cudaMallocs {a1 - a0} reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB", end=" ")
    print(f"rep{rep}: {dt:.3f}s {s.compute_runs / dt / 1e6:.1f}M/s setup {s.device_transfer.get('setup_s', 0):.3f}s "
          f"first_final {log[0][0] - t0:.3f}s "
          f"admitting rounds {adm} max gap {max(gaps) * 1e3:.1f}ms rounds {len(log)}", flush=True)
dt, lg, t0 = max(runs, key=lambda r: r[0])
print("slowest run, finalize times (ms):", [round((x[0] - t0) * 1e3) for x in lg])
print("slowest run, speculation depth:", [x[2] for x in lg])
