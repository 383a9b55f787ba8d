"""The long inputs of a round (GPU): retired count, status, the scalar
arguments and the mutation trace of every input above a retired threshold.
Usage: python tools/long_inputs.py [workload] [R] [threshold]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import collections
import numpy as np
from paper_2603_05725_b200.engine import DeviceCampaign
from paper_2603_05725_b200.lowering import VERDICT
from paper_2603_05725_b200.workloads import load

name = sys.argv[1] if len(sys.argv) > 1 else "matmul"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
thr = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
dc = DeviceCampaign(load(name), master_seed=11)
dc.run_round(1, R)
res = dc.run_round(1 + R, R)
S = res.slot
v = S.verdicts[:S.n * VERDICT.itemsize].cpu().numpy().view(VERDICT)
ret = v["retired"].astype(np.int64)
idx = np.nonzero(ret >= thr)[0]
print(f"{name}: {len(idx)} of {S.n} inputs retire >= {thr}; their share of retired: "
      f"{ret[idx].sum() / ret.sum():.1%}; max {ret.max():,}")
hist = collections.Counter(int(np.log2(max(r, 1))) for r in ret)
print("log2(retired) histogram:", dict(sorted(hist.items())))
ns = (v["where"] >> 9).astype(np.int64)
rer = (v["where"] >> 8) & 1
print(f"sequential re-runs (conflicts) among them: {int(rer[idx].sum())}")
order = idx[np.argsort(-ns[idx])][:40]          # slowest first
tcs = dc.child_testcases([int(i) for i in order], S)
for i, tc in zip(order, tcs):
    scal = [a.value if hasattr(a, "value") else f"arr{len(a.data)}" for a in tc.args]
    ops = [(o.kind, o.arg) for o in tc.trace]
    print(f"  it={int(S.it0 + i)} ms={ns[i] / 1e6:7.2f} rerun={int(rer[i])} retired={int(ret[i]):>9,} "
          f"status={int(v['status'][i])} args={scal} ops={ops}")
