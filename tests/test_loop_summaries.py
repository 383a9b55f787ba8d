"""Loop summaries of the specialized kernel (csrc/jit.cu analyse_cycle): long
pure-register loops are skipped in closed form, then finished instruction by
instruction.  Goldens from the REAL reference (tests/golden/make_golden.py loops):
explicit inputs whose loops exit by ==, !=, <= and > compares of wrapping i32
induction variables, or exhaust the budget at every position of the loop body
(budgets 10^6 + k), and whole batched campaigns of the two loop kernels with a
50,000-instruction budget through every execution mode (bulk pass with
deferral, group-parallel bulk, no deferral)."""

import ctypes
import hashlib
import sys
from pathlib import Path

import pytest

from conftest import golden, workload_manifest
from paper_2603_05725_b200.coverage import build_report, report_to_rec
from paper_2603_05725_b200.testcase import parse_testcase, serialize_testcase

REPO = Path(__file__).resolve().parent.parent


def _manifest(kern):
    from paper_2603_05725_b200.manifest import harness_from_text
    d = golden("ref_loops.json")
    return harness_from_text(d["manifests"][kern], d["kernel"], f"loops/{kern}.man")


def _source(m):
    sys.path.insert(0, str(REPO / "tools"))
    import jit_check
    rc, _, src = jit_check.check(m)
    assert rc == 0, src[:2000]
    return src


def test_summaries_generated_for_pure_register_cycles():
    """matmul's row loop (rows -> cols -> next_row with N <= 0) is summarized at
    both of its check blocks (the rotation starting at `cols` carries r15 = 0 as
    a guarded stable register); cycles through loads are not."""
    src = _source(workload_manifest("matmul"))
    assert src.count("// loop summary: blocks 1 2 3 8") == 2     # PAR and sequential window paths
    assert src.count("// loop summary: blocks 3 8 1 2") == 2
    assert "r15 == 0x00000000u" in src
    assert "blocks 5 6" not in src and "blocks 3 4 5 7" not in src
    for k in ("spin", "spin2"):
        assert src_count(_source(_manifest(k))) >= 4


def src_count(src):
    return src.count("// loop summary:")


@pytest.mark.gpu
@pytest.mark.parametrize("kern", ["spin", "spin2", "matmul"])
def test_loop_inputs_match_reference(cuda_ok, kern):
    from paper_2603_05725_b200.engine import DeviceCampaign
    d = golden("ref_loops.json")
    m = workload_manifest("matmul") if kern == "matmul" else _manifest(kern)
    recs = d["inputs"][kern]
    for budget in d["budgets"]:
        rs = [r for r in recs if r["budget"] == budget]
        dc = DeviceCampaign(m, master_seed=1, budget=budget, diff_readback=True)
        outs = dc.execute_testcases([parse_testcase(r["testcase"])[0] for r in rs], iteration0=1)
        for i, (out, r) in enumerate(zip(outs, rs)):
            where = (budget, i, r["testcase"].splitlines()[-5:])
            assert out["status"] == r["status"], where
            assert out["retired"] == r["retired"], where
            assert (out["report"].to_line() if out["report"] else None) == r["report"], where
            assert out["edges"] == r["edges"], where
            assert {k: v.hex() for k, v in out["readouts"].items()} == r["readouts"], where
        dc.close()


def _digest(tc):
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


@pytest.mark.gpu
@pytest.mark.parametrize("kern", ["spin", "spin2"])
@pytest.mark.parametrize("mode", ["default", "group", "nodefer", "nosum"])
def test_loop_campaigns_match_reference(cuda_ok, kern, mode, monkeypatch):
    from paper_2603_05725_b200.engine import DeviceCampaign
    d = golden("ref_loops.json")
    cfg = d["campaign_config"]
    ref = d["campaigns"][kern]
    kw = {}
    if mode == "group":
        monkeypatch.setenv("SFG_BULK_GROUP", "32")
    if mode == "nodefer":
        kw["soft_cap"] = 0
    if mode == "nosum":
        monkeypatch.setenv("SFG_LOOPSUM", "0")
    dc = DeviceCampaign(_manifest(kern), master_seed=cfg["master_seed"], budget=cfg["budget"], **kw)
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
    if mode != "nosum":
        nb = dc.L.sfg_program_jit_source(dc.h, None, 0)
        buf = ctypes.create_string_buffer(nb + 1)
        dc.L.sfg_program_jit_source(dc.h, buf, nb + 1)
        assert "// loop summary:" in buf.value.decode()
    dc.close()


def test_nest_summary_generated_for_matmul_rows():
    """matmul's row loop with its cols / inner loops, loads of A and B and stores of
    C is a nest summary (csrc/jit.cu analyse_nest): one induction register (the
    row), the row test as closed-form exit, the A / C address guards and the
    load-vs-store record guards, all conditional on the block having run."""
    src = _source(workload_manifest("matmul"))
    assert src.count("// nest summary: blocks 1 2 3 4 5 6 7 8") == 1
    assert "(uint32_t)(r14 * r5)" in src and "(uint32_t)(r14 * r3)" in src
    assert "pt0 != pt2" in src and "pt1 != pt2" in src


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["default", "nonest"])
def test_nest_inputs_match_reference(cuda_ok, mode, monkeypatch):
    """matmul row loops with loads and stores (zero / wrapping leading dimensions)
    to the budget at every position of a row trip (budgets 10^6 + 97 k), to the
    row exit, and with failing guards, equal the REAL reference's records
    (tests/golden/ref_nests.json): status, retired, report, edges, readouts."""
    from paper_2603_05725_b200.engine import DeviceCampaign
    if mode == "nonest":
        monkeypatch.setenv("SFG_NESTSUM", "0")
    d = golden("ref_nests.json")
    m = workload_manifest("matmul")
    for budget in d["budgets"]:
        rs = [r for r in d["records"] if r["budget"] == budget]
        dc = DeviceCampaign(m, master_seed=1, budget=budget, diff_readback=True)
        # each input alone at iteration 1, as the reference ran it (reports carry the iteration)
        outs = [dc.execute_testcases([parse_testcase(r["testcase"])[0]], iteration0=1)[0] for r in rs]
        for i, (out, r) in enumerate(zip(outs, rs)):
            where = (budget, i, d["inputs"][i])
            assert out["status"] == r["status"], where
            assert out["retired"] == r["retired"], where
            assert (out["report"].to_line() if out["report"] else None) == r["report"], where
            assert out["edges"] == r["edges"], where
            assert {k: v.hex() for k, v in out["readouts"].items()} == r["readouts"], where
        dc.close()


@pytest.mark.gpu
def test_array_alias_masks_for_matmul(cuda_ok):
    """jit.cu array_masks on C2 matmul: A and B are never stored (read from the
    parent's payload in place when unmutated), C is never loaded (not built)."""
    from paper_2603_05725_b200.engine import DeviceCampaign
    dc = DeviceCampaign(workload_manifest("matmul"), master_seed=1)
    nb = dc.L.sfg_program_jit_source(dc.h, None, 0)
    buf = ctypes.create_string_buffer(nb + 1)
    dc.L.sfg_program_jit_source(dc.h, buf, nb + 1)
    src = buf.value.decode()
    assert "#define SFG_RO_ARGS 3u" in src and "#define SFG_WO_ARGS 4u" in src
    dc.close()
