"""Pin the CPU oracle to the real reference (golden fixtures) and to numpy."""

import hashlib
import random

import numpy as np
import pytest

from conftest import bench_manifest, bench_names, golden, trigger_ops
from oracle import loop as ol
from oracle.mutate import apply_trace
from oracle.rng import OracleStream
from paper_2603_05725_b200.coverage import CoverageMap, build_report, report_to_rec
from paper_2603_05725_b200.testcase import parse_testcase, serialize_testcase


def _digest(tc):
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


def _edges(cov):
    return {k: sorted([list(e) + [c] for e, c in v.items()]) for k, v in cov.edge_counts.items() if v}


def test_rng_matches_numpy_generator():
    rr = random.Random(7)
    for _ in range(200):
        seed, sid = rr.randrange(1 << 64), rr.randrange(1 << 64)
        g = np.random.Generator(np.random.Philox(key=np.array([seed, sid], dtype=np.uint64)))
        o = OracleStream(seed, sid)
        for _ in range(40):
            k = rr.randrange(4)
            if k == 0:
                assert float(g.random()) == o.random()
            elif k == 1:
                lo = rr.randrange(-500, 500)
                hi = lo + rr.choice([1, 2, 3, 5, 8, 256, 1 << 23, 1 << 31, 1 << 32, (1 << 32) + 3, 1 << 50])
                assert int(g.integers(lo, hi)) == o.integers(lo, hi)
            elif k == 2:
                assert int(g.integers(0, 1 << 64, dtype=np.uint64)) == o.u64()
            else:
                assert int(g.integers(0, 1 << 32)) == o.integers(0, 1 << 32)


@pytest.mark.parametrize("name", bench_names())
def test_variants_land_their_class(name):
    ref = golden("ref_variants.json")
    for variant in ("spatial_oob", "temporal_uaf", "space_mismatch", "provenance_escape"):
        m = bench_manifest(name, variant)
        expected, ops = trigger_ops(name, variant)
        tc = apply_trace(m.seed(0), ops)
        cov = CoverageMap.for_program(m.program)
        out, _ = ol.execute_once(m, tc, coverage=cov)
        want = ref[f"{name}/{variant}"]
        assert out.status == want["status"] == "finding"
        assert out.report.bug_class.value == expected == want["expected"]
        assert out.report.to_line() == want["report"]
        assert out.retired == want["retired"]
        assert _edges(cov) == want["edges"]


@pytest.mark.parametrize("name", bench_names())
def test_sampled_inputs_bit_exact(name):
    from oracle.memory import Image
    m = bench_manifest(name)
    img = Image()
    run = ol.Runner(m, img, diff_readback=True)
    run.run("init", m.seed(1), iteration=0)
    run.mark_baseline()
    snap = img.snapshot()
    for i, rec in enumerate(golden("ref_sampled.json")[name]):
        tc, _ = parse_testcase(rec["testcase"])
        img.restore(snap)
        run.reset()
        cov = CoverageMap.for_program(m.program)
        out = run.run("compute", tc, coverage=cov, iteration=i + 1)
        assert out.status == rec["status"], i
        assert (out.report.to_line() if out.report else None) == rec["report"], i
        assert {k: v.hex() for k, v in out.readouts.items()} == rec["readouts"], i
        assert out.retired == rec["retired"]
        assert _edges(cov) == rec["edges"]


@pytest.mark.parametrize("name", bench_names())
def test_batched_contract_matches_reference(name):
    data = golden("ref_batched.json")
    cfg = data["config"]
    assert data["keybase"] == ol.KEYBASE
    ref = data["runs"][name]
    m = bench_manifest(name)
    res = ol.batched_loop(m, master_seed=cfg["master_seed"], iterations=cfg["iterations"],
                          round_size=cfg["round_size"])
    assert len(res.records) == len(ref["records"])
    for got, want in zip(res.records, ref["records"]):
        assert got["parent"] == want["parent"], got["it"]
        assert _digest(got["child"]) == want["child"], got["it"]
        assert str(got["child"].rng_seed) == want["rng_seed"]
        assert [op.encode() for op in got["child"].trace] == want["trace"]
        assert got["status"] == want["status"]
        assert got["report"] == want["report"], got["it"]
        assert got["retired"] == want["retired"]
        assert got["allocs"] == want["allocs"]
        assert got["edges"] == want["edges"]
        assert got["admitted"] == want["admitted"]
    assert res.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(res.coverage)) == ref["coverage"]
    assert [_digest(e.tc) for e in res.corpus] == ref["corpus"]


@pytest.mark.parametrize("key", sorted(golden("ref_fuzzloop.json")))
def test_sequential_loop_matches_reference_fuzz_loop(key):
    name, seed, iters = key.split("/")
    want = golden("ref_fuzzloop.json")[key]
    m = bench_manifest(name)
    res = ol.sequential_loop(m, master_seed=int(seed), iterations=int(iters), keep_records=False,
                             **want["kw"])
    assert res.findings.render_text() == want["findings"]
    assert report_to_rec(build_report(res.coverage)) == want["coverage_rec"]
    assert sorted(f"{e.tc.id}.tc" for e in res.corpus) == want["corpus"]
    assert f"stop={res.stop_reason}" in want["summary"]
    assert f"compute_runs={res.executed}" in want["summary"]


@pytest.mark.parametrize("stem", ["matmul", "vadd", "ctxchain", "structcfg"])
def test_workloads_batched_matches_reference(stem):
    """C1-C4 synthetic targets (workloads/*.man): the oracle's batched driver vs
    the reference's own functions driven the same way (make_golden.py workloads)."""
    from conftest import workload_case
    ref = golden("ref_workloads.json")[stem]
    m, kw, R, iters = workload_case(stem)
    res = ol.batched_loop(m, master_seed=11, iterations=iters, round_size=R, **kw)
    assert len(res.records) == len(ref["records"])
    for got, want in zip(res.records, ref["records"]):
        assert got["parent"] == want["parent"], got["it"]
        assert _digest(got["child"]) == want["child"], got["it"]
        assert got["report"] == want["report"], got["it"]
        assert got["retired"] == want["retired"], got["it"]
        assert got["edges"] == want["edges"], got["it"]
        assert got["admitted"] == want["admitted"], got["it"]
    assert res.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(res.coverage)) == ref["coverage"]
    assert [_digest(e.tc) for e in res.corpus] == ref["corpus"]
