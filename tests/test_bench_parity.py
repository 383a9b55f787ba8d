"""Parity at the benchmarked configurations (tests/golden/make_golden_bench.py).

C2: the bench's own setup -- workloads/matmul.man, master_seed 11, rounds of
R = 2^20, 24 rounds in flight, the default soft cap (long inputs deferred to
the tail pass), sfg_order on -- against the REAL reference's batched-round
records: every input of round 1 (per-1024-input block hashes of the records,
the first 20,000 records compared field by field), the campaign state after
round 1 (findings.txt, coverage.rec, corpus), and the first 4,096 inputs of
round 2 (records are prefix-consistent within a round).

C5: the dot + amax + rotm mix at R = 2^14, two full rounds each.
"""

import gzip
import hashlib
import json
from functools import lru_cache

import pytest

from conftest import GOLDEN, bench_manifest, workload_manifest
from paper_2603_05725_b200.coverage import build_report, report_to_rec
from paper_2603_05725_b200.testcase import serialize_testcase

pytestmark = pytest.mark.gpu


@lru_cache(maxsize=None)
def _gz(name):
    with gzip.open(GOLDEN / name, "rt") as f:
        return json.load(f)


def _digest(tc):
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


def golden_record(g) -> dict:
    """A device record in the reference fixture's shape (make_golden_bench.campaign)."""
    c = g["child"]
    return {"it": g["it"], "parent": g["parent"], "child": _digest(c), "rng_seed": str(c.rng_seed),
            "trace": [op.encode() for op in c.trace], "status": g["status"], "retired": g["retired"],
            "allocs": g["allocs"], "edges": g["edges"], "admitted": g["admitted"], "report": g["report"]}


def record_hash(rec) -> str:
    return hashlib.sha256(json.dumps(rec, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def block_hashes(recs, block):
    out = []
    for b in range(0, len(recs), block):
        h = hashlib.sha256()
        for r in recs[b:b + block]:
            h.update(record_hash(r).encode())
        out.append(h.hexdigest()[:32])
    return out


def _check_rounds(dc, rounds_ref, block, depth):
    """Run the campaign over the fixture's rounds; compare each round's records and
    the campaign state after it."""
    R = rounds_ref[0]["n"]
    it_stop = 1 + sum(r["n"] for r in rounds_ref)
    seen = []

    def on_round(res):
        recs = [golden_record(g) for g in dc.round_records(res)]
        seen.append({"it0": res.it0, "n": len(recs), "recs": recs, "findings": dc.findings.render_text(),
                     "coverage": report_to_rec(build_report(dc.coverage_map())),
                     "corpus": [_digest(e[0]) for e in dc.host_entries], "next_alloc_id": dc.next_alloc_id})

    dc.run_rounds(1, it_stop, R, depth=depth, on_round=on_round)
    assert len(seen) == len(rounds_ref)
    for got, want in zip(seen, rounds_ref):
        assert (got["it0"], got["n"]) == (want["it0"], want["n"])
        for g, w in zip(got["recs"], want["records"]):
            assert g == w, g["it"]
        gb = block_hashes(got["recs"], block)
        bad = [k for k, (x, y) in enumerate(zip(gb, want["blocks"])) if x != y]
        assert len(gb) == len(want["blocks"]) and not bad, f"blocks differ: {bad[:8]}"
        assert got["findings"] == want["findings"]
        assert got["coverage"] == want["coverage"]
        assert got["corpus"] == want["corpus"]
        assert got["next_alloc_id"] == want["next_alloc_id"]
        assert [r["it"] for r in got["recs"] if r["admitted"]] == want["admitted"]


@pytest.mark.parametrize("mode", ["default", "lowcap", "plain"])
def test_c2_bench_configuration_matches_reference(cuda_ok, mode, monkeypatch):
    """default: bench.py's own setup.  lowcap: a 2,048-instruction soft cap sends
    every longer input through the group-parallel long-input pass (nest summaries
    under conflict tags).  plain: no nest summaries and no equal-input schedule."""
    from paper_2603_05725_b200.engine import DeviceCampaign
    ref = _gz("ref_bench_c2.json.gz")
    cfg = ref["config"]
    assert cfg["round_size"] == 1 << 20      # bench.py's default --round
    kw = {}
    if mode == "lowcap":
        kw["soft_cap"] = 2048
    if mode == "plain":
        monkeypatch.setenv("SFG_NESTSUM", "0")
        monkeypatch.setenv("SFG_GROUP_DUPS", "0")
    dc = DeviceCampaign(workload_manifest("matmul"), master_seed=cfg["master_seed"], **kw)   # bench.py's defaults
    _check_rounds(dc, ref["rounds"], ref["block"], depth=24)
    dc.close()


@pytest.mark.parametrize("name", ["dot", "amax", "rotm"])
def test_c5_mix_two_rounds_match_reference(cuda_ok, name):
    from paper_2603_05725_b200.engine import DeviceCampaign
    ref = _gz("ref_bench_c5.json.gz")
    dc = DeviceCampaign(bench_manifest(name), master_seed=ref["config"]["master_seed"])
    _check_rounds(dc, ref["runs"][name], ref["block"], depth=8)
    dc.close()
