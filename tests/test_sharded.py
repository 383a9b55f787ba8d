"""Multi-GPU round sharding: the per-round merge.

CPU (gloo, world size 2): the RoundComm collectives and the merge algebra the
triage kernels implement -- per-rank partials (first hitter per edge = MIN,
counts = SUM) merged across ranks reproduce the reference's admissions and
campaign map on its own golden records.

GPU (gloo, 2 ranks sharing cuda:0): a sharded campaign through the product
kernels equals the single-rank campaign and the reference golden records.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import REPO, bench_manifest, golden
from paper_2603_05725_b200.shard import owner_of, shard_bounds

NONE = 0x7FFFFFFF


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_partition():
    for n in (0, 1, 5, 64, 100, 65536):
        for w in (1, 2, 3, 4, 8):
            got = [shard_bounds(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            for i in range(0, n, max(1, n // 7)):
                lo, hi = got[owner_of(i, n, w)]
                assert lo <= i < hi


def _edge_index(records):
    names = sorted({(k, a, b) for r in records for k, es in r["edges"].items() for a, b, _ in es})
    return {e: j for j, e in enumerate(names)}


def _merge_worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2603_05725_b200.shard import RoundComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = RoundComm()
    # collective primitives
    t = torch.tensor([5 + rank, NONE, 3 - rank], dtype=torch.int32)
    comm.all_reduce(t, "min")
    assert t.tolist() == [5, NONE, 2]
    u = torch.tensor([1, 10 * rank], dtype=torch.int64)
    comm.all_reduce(u, "sum")
    assert u.tolist() == [world, 10 * sum(range(world))]
    g = comm.all_gather(torch.tensor([rank, rank * 2], dtype=torch.int64))
    assert g.tolist() == [[r, 2 * r] for r in range(world)]
    assert comm.all_gather_object({"r": rank}) == [{"r": r} for r in range(world)]

    # merge algebra over the reference's golden batched records
    data = golden("ref_batched.json")
    R = data["config"]["round_size"]
    ok = True
    for name in ("amax", "rotm", "dot"):
        recs = data["runs"][name]["records"]
        eidx = _edge_index(recs)
        E = len(eidx)
        ghit = np.zeros(E, bool)
        total = torch.zeros(E, dtype=torch.int64)
        for r0 in range(0, len(recs), R):
            rnd = recs[r0:r0 + R]
            lo, hi = comm.bounds(len(rnd))
            first = torch.full((E,), NONE, dtype=torch.int32)
            delta = torch.zeros(E, dtype=torch.int64)
            for i in range(lo, hi):
                for k, es in rnd[i]["edges"].items():
                    for a, b, c in es:
                        e = eidx[(k, a, b)]
                        first[e] = min(int(first[e]), i)
                        delta[e] += c
            comm.all_reduce(first, "min")
            comm.all_reduce(delta, "sum")
            adm = []
            for i in range(lo, hi):
                r = rnd[i]
                hit = [eidx[(k, a, b)] for k, es in r["edges"].items() for a, b, _ in es]
                adm.append(r["report"] is None and r["it"] != 1
                           and any(not ghit[e] and int(first[e]) == i for e in hit))
            merged = [a for part in comm.all_gather_object(adm) for a in part]
            ok &= merged == [r["admitted"] for r in rnd]
            total += delta
            ghit |= (total > 0).numpy()
        want = np.zeros(E, np.int64)
        for r in recs:
            for k, es in r["edges"].items():
                for a, b, c in es:
                    want[eidx[(k, a, b)]] += c
        ok &= bool((total.numpy() == want).all())
    if rank == 0:
        with open(out_path, "w") as f:
            f.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


def test_round_merge_gloo_world2():
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.start_processes(_merge_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
        assert open(out).read() == "ok"


# ---------------------------------------------------------------- GPU: the product path, sharded


def _campaign_worker(rank, world, port, out_path, which, backend="gloo"):
    import hashlib
    import json
    import sys
    sys.path.insert(0, str(REPO / "tests"))
    import torch.distributed as dist
    from paper_2603_05725_b200.coverage import build_report, report_to_rec
    from paper_2603_05725_b200.engine import DeviceCampaign
    from paper_2603_05725_b200.shard import RoundComm
    from paper_2603_05725_b200.testcase import serialize_testcase
    # gloo: every rank on cuda:0 (collectives staged through host memory); nccl: one GPU per rank
    torch.cuda.set_device(rank if backend == "nccl" else 0)
    if world > 1:
        dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    if which == "matmul":
        from conftest import workload_manifest
        m, R, iters = workload_manifest("matmul"), 100, 300
    else:
        m, R, iters = bench_manifest(which), 128, 600
    dc = DeviceCampaign(m, master_seed=11, comm=RoundComm())
    dc.run_rounds(1, iters + 1, R, depth=3)
    dig = [hashlib.sha256(serialize_testcase(e[0], with_id=False).encode()).hexdigest()[:32] for e in dc.host_entries]
    res = {"findings": dc.findings.render_text(), "coverage": report_to_rec(build_report(dc.coverage_map())),
           "corpus": dig}
    dc.close()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(res, f)
    if world > 1:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["amax", "matmul"])
def test_sharded_campaign_equals_reference(cuda_ok, which):
    import json
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.json")
        mp.start_processes(_campaign_worker, args=(2, _free_port(), out, which), nprocs=2, start_method="spawn")
        got = json.load(open(out))
    ref = golden("ref_workloads.json")["matmul"] if which == "matmul" else golden("ref_batched.json")["runs"][which]
    assert got["findings"] == ref["findings"]
    assert got["coverage"] == ref["coverage"]
    assert got["corpus"] == ref["corpus"]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("which", ["amax", "matmul"])
def test_nccl_sharded_campaign_equals_reference(cuda_ok, which, world):
    """The NCCL path itself (one process per GPU, NCCL all-reduce / all-gather of the
    per-round partials): the sharded campaign equals the reference golden records
    for every GPU count the box has (skipped on a one-GPU box)."""
    import json
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.json")
        mp.start_processes(_campaign_worker, args=(world, _free_port(), out, which, "nccl"), nprocs=world,
                           start_method="spawn")
        got = json.load(open(out))
    ref = golden("ref_workloads.json")["matmul"] if which == "matmul" else golden("ref_batched.json")["runs"][which]
    assert got["findings"] == ref["findings"]
    assert got["coverage"] == ref["coverage"]
    assert got["corpus"] == ref["corpus"]
