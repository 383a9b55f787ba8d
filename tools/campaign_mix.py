"""C5 on one GPU: a 1e9-exec campaign over the harness mix
dot + amax + rotm (the reference's bundled benchmarks, tests/golden/bench_assets.json),
master_seed 11, fixed global round size, one campaign per harness back to back.
Prints per-harness execs/s, findings / coverage / corpus digests (GPU only).
Usage: python tools/campaign_mix.py [total_execs] [R] [depth]"""
import hashlib, json, sys, time
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import paper_2603_05725_b200  # noqa: F401
import torch
from conftest import bench_manifest
from paper_2603_05725_b200.coverage import build_report, report_to_rec
from paper_2603_05725_b200.engine import DeviceCampaign

total = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
D = int(sys.argv[3]) if len(sys.argv) > 3 else 16
names = ["dot", "amax", "rotm"]
per = total // len(names) // R * R
out = {"total_execs": 0, "round_size": R, "depth": D, "harnesses": {}}
t_all = time.perf_counter()
for name in names:
    dc = DeviceCampaign(bench_manifest(name), master_seed=11)
    dc.reserve(D, R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dc.run_rounds(1, 1 + per, R, depth=D)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ex = sum(r.executed for r in res)
    cov = report_to_rec(build_report(dc.coverage_map()))
    out["harnesses"][name] = {
        "execs": ex, "seconds": dt, "execs_per_s": ex / dt, "findings_unique": len(dc.findings),
        "findings_sha256": hashlib.sha256(dc.findings.render_text().encode()).hexdigest()[:16],
        "coverage_sha256": hashlib.sha256(cov.encode()).hexdigest()[:16], "corpus": len(dc.host_entries)}
    out["total_execs"] += ex
    print(name, json.dumps(out["harnesses"][name]), flush=True)
    dc.close()
    del dc, res
out["seconds"] = time.perf_counter() - t_all
out["execs_per_s"] = out["total_execs"] / out["seconds"]
print(json.dumps(out))
