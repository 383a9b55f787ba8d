"""Objects of the reference package (``simt_forge``) in and out of this framework.

A caller of the reference hands its own objects to :func:`campaign.fuzz_loop`:
a ``simt_forge.campaign.HarnessManifest`` (from ``load_harness`` or the bundled
benchmarks), a ``simt_forge.campaign.CampaignConfig`` and ``simt_forge``
``TestCase`` values.  They are recognised by shape (duck typing: this package
never imports the reference) and converted through their public fields and enum
``.value`` strings:

* a manifest is re-read from its canonical text (``normalized`` +
  ``program_text``, campaign.py:99-120), so digests are identical;
* a reference ``CampaignConfig`` (campaign.py:609-625) becomes this package's
  config with ``discipline="sequential"``: the reference object carries no
  round / discipline fields, so it asks for the reference ``fuzz_loop``'s own
  semantics, which the sequential discipline reproduces exactly;
* test cases, values and mutation ops keep their fields (ids are equal).

``CampaignSummary.to_reference(simt_forge_module)`` goes the other way: the
findings, coverage and corpus as the reference's own types, for callers that
keep using ``simt_forge`` APIs on the results.
"""

from __future__ import annotations

from dataclasses import fields

from .findings import BugClass, BugReport
from .sir import MemSpace
from .testcase import ArrayValue, FloatValue, IntValue, MutationOp, TestCase


def _is_ours(obj) -> bool:
    return type(obj).__module__.startswith(__package__ + ".")


def as_manifest(m):
    """This package's HarnessManifest for ``m`` (ours, or the reference's)."""
    from .manifest import HarnessManifest, harness_from_text
    if isinstance(m, HarnessManifest):
        return m
    if not (hasattr(m, "normalized") and hasattr(m, "program_text")):
        raise TypeError(f"not a harness manifest: {type(m).__name__}")
    return harness_from_text(m.normalized, m.program_text, getattr(m, "path", "harness.man"),
                             getattr(m, "program_path", None))


def as_value(v):
    if _is_ours(v):
        return v
    kind = type(v).__name__
    if kind == "IntValue":
        return IntValue(int(v.value))
    if kind == "FloatValue":
        return FloatValue(int(v.bits))
    if kind == "ArrayValue":
        return ArrayValue(bytes(v.data), str(v.elem), tuple(int(e) for e in v.extents), MemSpace(v.space.value),
                          int(v.base_offset), None if v.size_override is None else int(v.size_override))
    raise TypeError(f"not a test-case value: {kind}")


def as_op(op):
    return op if _is_ours(op) else MutationOp(str(op.kind), int(op.arg), tuple((str(k), str(x)) for k, x in op.params))


def as_testcase(tc):
    """This package's TestCase for ``tc`` (ours, or the reference's): same fields, same id."""
    if isinstance(tc, TestCase):
        return tc
    return TestCase(tuple(as_value(v) for v in tc.args), int(tc.rng_seed), tc.parent_id,
                    tuple(as_op(o) for o in tc.trace))


def as_config(cfg):
    """This package's CampaignConfig for ``cfg``; a reference config selects the
    reference fuzz_loop semantics (discipline "sequential")."""
    from .baseline import MemConfig
    from .campaign import CampaignConfig
    from .engine import MutationConfig
    if isinstance(cfg, CampaignConfig):
        return cfg
    kw = {}
    for f in fields(CampaignConfig):
        if hasattr(cfg, f.name):
            kw[f.name] = getattr(cfg, f.name)
    if "mem_config" in kw and not isinstance(kw["mem_config"], MemConfig):
        mc = kw["mem_config"]
        kw["mem_config"] = MemConfig(**{f.name: getattr(mc, f.name) for f in fields(MemConfig) if hasattr(mc, f.name)})
    if "mutation" in kw and not isinstance(kw["mutation"], MutationConfig):
        mu = kw["mutation"]
        kw["mutation"] = MutationConfig(**{f.name: getattr(mu, f.name) for f in fields(MutationConfig)
                                           if hasattr(mu, f.name)})
    sbc = kw.get("stop_bug_class")
    if sbc is not None and not isinstance(sbc, (str, BugClass)):
        kw["stop_bug_class"] = BugClass(sbc.value)
    kw.setdefault("discipline", "sequential")
    return CampaignConfig(**kw)


# ---- results back as reference objects --------------------------------------------
def _mod(sf, name):
    import importlib
    return importlib.import_module(f"{sf.__name__}.{name}")


def report_to_reference(rep: BugReport, sf):
    san = _mod(sf, "sanitizer")
    mem = _mod(sf, "kernel_ir").MemSpace
    return san.BugReport(san.BugClass(rep.bug_class.value), rep.kernel, rep.iid, rep.ctaid, rep.tid, rep.address,
                         rep.width, rep.is_store, None if rep.declared_space is None else mem(rep.declared_space.value),
                         rep.mechanism, rep.shadow_code, rep.provenance, rep.alloc_id, rep.alloc_label,
                         rep.alloc_base, rep.alloc_size, rep.alloc_state, rep.iteration)


def testcase_to_reference(tc: TestCase, sf):
    mu = _mod(sf, "mutation")
    mem = _mod(sf, "kernel_ir").MemSpace

    def val(v):
        if isinstance(v, IntValue):
            return mu.IntValue(v.value)
        if isinstance(v, FloatValue):
            return mu.FloatValue(v.bits)
        return mu.ArrayValue(v.data, v.elem, v.extents, mem(v.space.value), v.base_offset, v.size_override)

    return mu.TestCase(tuple(val(v) for v in tc.args), tc.rng_seed, tc.parent_id,
                       tuple(mu.MutationOp(o.kind, o.arg, o.params) for o in tc.trace))


def summary_to_reference(summary, sf, program):
    """(FindingsLog, CoverageMap, Corpus) of the reference package ``sf`` (the
    ``simt_forge`` module) for a summary of this package; ``program`` is the
    reference Program the coverage describes (``reference_manifest.program``)."""
    findings = _mod(sf, "sanitizer").FindingsLog()
    for rep in summary.findings.reports():
        r = report_to_reference(rep, sf)
        findings.add(r)
        findings._counts[r.dedupe_key] = summary.findings.count(rep.dedupe_key)   # hit counts, not re-added
    cov = _mod(sf, "coverage").CoverageMap.for_program(program)
    for k, counts in summary.coverage.edge_counts.items():
        for (s, d), c in counts.items():
            cov.record_edge(k, s, d, c)
        if summary.coverage.entered[k]:
            cov.record_launch(k)
    corpus = _mod(sf, "campaign").Corpus()
    for e in summary.corpus.entries:
        tc = testcase_to_reference(e.tc, sf)
        if e.is_seed:
            corpus.add_seed(tc)
        else:
            corpus.admit(tc, e.admitted_iteration)
    return findings, cov, corpus
