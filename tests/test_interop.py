"""The reference's own objects through this package's API (interop.py): a
``simt_forge`` HarnessManifest / CampaignConfig / TestCase in, and the results
back as ``simt_forge`` FindingsLog / CoverageMap / Corpus.  The reference is
imported from /root/reference (build container) or baseline/_ref (the offline
install that travels to the GPU box); the tests skip when neither exists."""

import sys
from pathlib import Path

import pytest

from conftest import golden

REPO = Path(__file__).resolve().parent.parent
for p in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (p / "simt_forge").exists():
        sys.path.insert(0, str(p))
        break
sf = pytest.importorskip("simt_forge")


def _ref():
    import simt_forge.bench as rb
    import simt_forge.campaign as rc
    import simt_forge.mutation as rm
    return rb, rc, rm


def test_reference_objects_convert_on_cpu():
    """Manifest digests, test-case ids and config fields survive the conversion."""
    from paper_2603_05725_b200.interop import as_config, as_manifest, as_testcase
    rb, rc, rm = _ref()
    from simt_forge.rng import Stream
    for name in ("dot", "rotm", "copy"):
        m = rb.get_benchmark(name).load()
        mine = as_manifest(m)
        assert (mine.digest, mine.program_digest) == (m.digest, m.program.digest)
        sched = rm.MutationSchedule()
        tc = m.seed(3)
        for k in range(20):
            tc = rm.mutate_testcase(tc, m.argspecs, sched, Stream(5, k))
            assert as_testcase(tc).id == tc.id
    cfg = as_config(rc.CampaignConfig(master_seed=7, iterations=99, stop_bug_class="SPATIAL_OOB"))
    assert (cfg.master_seed, cfg.iterations, cfg.discipline) == (7, 99, "sequential")


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(golden("ref_fuzzloop.json")))
def test_reference_objects_through_fuzz_loop(cuda_ok, key, tmp_path):
    """fuzz_loop(simt_forge manifest, simt_forge CampaignConfig) reproduces the
    reference fuzz_loop (its config selects the sequential discipline), and the
    results convert back to simt_forge types with identical renderings."""
    from paper_2603_05725_b200.campaign import fuzz_loop
    rb, rc, rm = _ref()
    import simt_forge.coverage as rcov
    want = golden("ref_fuzzloop.json")[key]
    name, seed, iters = key.split("/")
    m = rb.get_benchmark(name).load()
    cfg = rc.CampaignConfig(master_seed=int(seed), iterations=int(iters), out_dir=tmp_path / "o", **want["kw"])
    s = fuzz_loop(m, cfg)
    assert s.to_rec() == want["summary"]
    findings, cov, corpus = s.to_reference(sf, m)
    assert isinstance(findings, sf.sanitizer.FindingsLog) and isinstance(corpus, rc.Corpus)
    assert findings.render_text() == want["findings"]
    assert rcov.report_to_rec(rcov.build_report(cov)) == want["coverage_rec"]
    assert sorted(e.tc.id + ".tc" for e in corpus.entries) == want["corpus"]
