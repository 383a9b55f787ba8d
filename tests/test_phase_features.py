"""Harness features beyond the bundled benchmarks, against the REAL reference
(tests/golden/make_golden.py features; campaign.py:483-561, 723-762):

* bufwrite   -- every exec stores >= 5 KB into an INIT (`buf:`) buffer: the
                per-input copy-on-write overlay of 256-byte chunks, grown (and the
                round re-run) when an input needs more chunks than it holds;
* initlaunch -- an INIT-phase launch over an INIT buffer and an array argument
                materialized in INIT (run once on the device, its results become
                the baseline every input starts from);
* termlaunch -- a TERM-phase launch that reports (iteration -1) and a double
                free that TERM skips;
* copyarg    -- COMPUTE `copy_in <buf> arg:N` of an array argument after a
                launch modified that argument (the test case's own bytes are
                copied, from a pristine copy in the work region).

Batched-round records (child, verdict line, retired, allocs, edges, admission),
findings, coverage and corpus; and reference `fuzz_loop` output directories
(discipline "sequential") including the TERM finding and its crash file.
"""

import hashlib

import pytest

from conftest import golden
from paper_2603_05725_b200.coverage import build_report, report_to_rec
from paper_2603_05725_b200.testcase import serialize_testcase

NAMES = ["bufwrite", "initlaunch", "termlaunch", "copyarg"]


def _manifest(name):
    from paper_2603_05725_b200.manifest import harness_from_text
    d = golden("ref_features.json")
    return harness_from_text(d["manifests"][name], d["kernel"], f"features/{name}.man")


def _digest(tc):
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


def test_features_lower_on_cpu():
    """Lowering accepts every feature (no LoweringError): copy_in from an array sets
    the pristine-copy mask, INIT-buffer stores get an overlay."""
    from paper_2603_05725_b200.baseline import MemConfig, build_baseline
    from paper_2603_05725_b200.engine import MutationConfig
    from paper_2603_05725_b200.lowering import Lowered
    for name in NAMES:
        m = _manifest(name)
        if name == "initlaunch":
            with pytest.raises(Exception, match="INIT-phase launches need the device"):
                build_baseline(m, m.seed(11), MemConfig())
            continue
        low = Lowered(m, build_baseline(m, m.seed(11), MemConfig()), mem=MemConfig(), mutation=MutationConfig(),
                      master_seed=11, budget=10 ** 6, window=256, recent_weight=4.0)
        if name == "copyarg":
            assert int(low.prog["copy_src_mask"]) == 1
        if name == "bufwrite":
            assert int(low.prog["ov_cap"]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", ["default", "group"])
def test_feature_campaigns_match_reference(cuda_ok, name, mode, monkeypatch):
    from paper_2603_05725_b200.engine import DeviceCampaign
    if mode == "group":
        monkeypatch.setenv("SFG_BULK_GROUP", "32")
    d = golden("ref_features.json")
    cfg = d["campaign_config"]
    ref = d["campaigns"][name]
    dc = DeviceCampaign(_manifest(name), master_seed=cfg["master_seed"])
    got = []
    dc.run_rounds(1, cfg["iterations"] + 1, cfg["round_size"], depth=3,
                  on_round=lambda res: got.extend(dc.round_records(res)))
    assert len(got) == len(ref["records"])
    for g, w in zip(got, ref["records"]):
        assert _digest(g["child"]) == w["child"], g["it"]
        assert (g["status"], g["report"], g["retired"], g["allocs"], g["edges"], g["admitted"]) == \
               (w["status"], w["report"], w["retired"], w["allocs"], w["edges"], w["admitted"]), g["it"]
    assert dc.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(dc.coverage_map())) == ref["coverage"]
    assert [_digest(e[0]) for e in dc.host_entries] == ref["corpus"]
    if name == "bufwrite":
        assert dc.ov_grows >= 2     # 5 KB per exec: 20 chunks > the initial 4
    dc.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_feature_fuzz_loops_match_reference(cuda_ok, name, tmp_path):
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    want = golden("ref_features.json")["fuzzloops"][name]
    d = tmp_path / "out"
    s = fuzz_loop(_manifest(name), CampaignConfig(master_seed=5, iterations=300, out_dir=d, round_size=64,
                                                  discipline="sequential"))
    assert (d / "findings.txt").read_text() == want["findings"]
    assert (d / "coverage.rec").read_text() == want["coverage_rec"]
    assert sorted(p.name for p in (d / "corpus").iterdir()) == want["corpus"]
    assert sorted(p.name for p in (d / "crashes").iterdir()) == want["crashes"]
    assert s.to_rec() == want["summary"]
