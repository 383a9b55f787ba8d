"""Debug probe (GPU): seqgen vs the one-thread walk on one harness at size n;
prints stats and where they first differ."""
import sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import numpy as np  # noqa: E402
from conftest import workload_manifest  # noqa: E402
from paper_2603_05725_b200.engine import CHILD, DeviceCampaign  # noqa: E402

m = workload_manifest(sys.argv[1] if len(sys.argv) > 1 else "matmul")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
dc = DeviceCampaign(m, master_seed=11, sequential=True)
dc.new_worker(0)
dc.run_rounds(1, 513, 512)
b = dc.seq_generate(513, n, parallel=True)
print("n", n, "stats", b[4], "mu", dc._seq_mu)
if n <= 200000:
    a = dc.seq_generate(513, n, parallel=False)
    ca = a[0].reshape(n, CHILD.itemsize)
    cb = b[0].reshape(n, CHILD.itemsize)
    bad = np.nonzero((ca != cb).any(1))[0]
    print("first differing child:", bad[:5], "of", len(bad))

if len(sys.argv) > 3:   # a pipelined campaign: per-round log
    import time
    import torch
    R = int(sys.argv[3])
    dc2 = DeviceCampaign(m, master_seed=11, sequential=True)
    dc2.new_worker(0)
    log = []
    t = time.perf_counter()
    dc2.run_rounds(1, 1 + 16 * R, R, depth=24, on_round=lambda r: log.append((r.it0, r.n, r.executed, r.n_admitted)))
    torch.cuda.synchronize()
    print("campaign", 16 * R, "in", round(time.perf_counter() - t, 3), "s; truncations", dc2.seq_truncations,
          "mu", round(dc2._seq_mu, 3))
    for x in log[:40]:
        print("  round", x)
