"""Scratch: print the first mismatching records between the GPU round and the oracle."""
import json, sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import torch
from paper_2603_05725_b200.manifest import harness_from_text
from paper_2603_05725_b200.engine import DeviceCampaign
from oracle.loop import batched_loop

name = sys.argv[1] if len(sys.argv) > 1 else "dot"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
a = json.loads((REPO / "tests/golden/bench_assets.json").read_text())[name]
m = harness_from_text(a["harness"], a["kernel"], f"{name}/harness.man")
dc = DeviceCampaign(m, master_seed=11)
res = dc.run_round(1, n)
got = dc.round_records(res)
ref = batched_loop(m, master_seed=11, iterations=n, round_size=n).records
bad = 0
for g, r in zip(got, ref):
    diffs = []
    if g["child"].id != r["child"].id:
        diffs.append(("child", [op.encode() for op in g["child"].trace], [op.encode() for op in r["child"].trace],
                      g["child"].rng_seed, r["child"].rng_seed))
    for k in ("parent", "status", "report", "retired", "allocs", "edges", "admitted"):
        if g[k] != r[k]:
            diffs.append((k, g[k], r[k]))
    if diffs:
        bad += 1
        if bad <= 6:
            print("it", g["it"], diffs)
print(f"{name}: {bad}/{len(got)} mismatching records")
