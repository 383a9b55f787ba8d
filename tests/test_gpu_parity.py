"""GPU parity: the sm_100a path (through the C ABI) vs the reference's golden
vectors and the CPU oracle, bit-exact."""

import hashlib

import numpy as np

import pytest

from conftest import bench_manifest, bench_names, golden, trigger_ops
from paper_2603_05725_b200.coverage import build_report, report_to_rec
from paper_2603_05725_b200.testcase import parse_testcase, serialize_testcase

pytestmark = pytest.mark.gpu

VARIANTS = ("spatial_oob", "temporal_uaf", "space_mismatch", "provenance_escape")


def _digest(tc):
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


@pytest.fixture(scope="module")
def engine_cls(cuda_ok):
    from paper_2603_05725_b200.engine import DeviceCampaign
    return DeviceCampaign


@pytest.mark.parametrize("name", bench_names())
def test_trigger_variants(engine_cls, name):
    from oracle.mutate import apply_trace
    ref = golden("ref_variants.json")
    for variant in VARIANTS:
        m = bench_manifest(name, variant)
        _, ops = trigger_ops(name, variant)
        tc = apply_trace(m.seed(0), ops)
        dc = engine_cls(m, master_seed=1)
        (out,) = dc.execute_testcases([tc])
        want = ref[f"{name}/{variant}"]
        assert out["status"] == want["status"]
        assert out["report"].to_line() == want["report"], variant
        assert out["retired"] == want["retired"]
        assert out["edges"] == want["edges"]
        dc.close()


@pytest.mark.parametrize("name", bench_names())
def test_sampled_inputs_readouts(engine_cls, name):
    m = bench_manifest(name)
    recs = golden("ref_sampled.json")[name]
    dc = engine_cls(m, master_seed=1, diff_readback=True)
    tcs = [parse_testcase(r["testcase"])[0] for r in recs]
    outs = dc.execute_testcases(tcs, iteration0=1)
    for i, (out, r) in enumerate(zip(outs, recs)):
        assert out["status"] == r["status"], i
        assert (out["report"].to_line() if out["report"] else None) == r["report"], i
        assert {k: v.hex() for k, v in out["readouts"].items()} == r["readouts"], i
        assert out["retired"] == r["retired"], i
        assert out["edges"] == r["edges"], i
    dc.close()


@pytest.mark.parametrize("name", bench_names())
def test_batched_rounds_match_reference(engine_cls, name):
    data = golden("ref_batched.json")
    cfg = data["config"]
    ref = data["runs"][name]
    m = bench_manifest(name)
    dc = engine_cls(m, master_seed=cfg["master_seed"])
    got = []
    it = 1
    while it <= cfg["iterations"]:
        n = min(cfg["round_size"], cfg["iterations"] - it + 1)
        res = dc.run_round(it, n)
        got += dc.round_records(res)
        it += n
    assert len(got) == len(ref["records"])
    for g, w in zip(got, ref["records"]):
        assert g["parent"] == w["parent"], g["it"]
        assert [op.encode() for op in g["child"].trace] == w["trace"], g["it"]
        assert str(g["child"].rng_seed) == w["rng_seed"], g["it"]
        assert _digest(g["child"]) == w["child"], g["it"]
        assert g["status"] == w["status"], g["it"]
        assert g["report"] == w["report"], g["it"]
        assert g["retired"] == w["retired"], g["it"]
        assert g["allocs"] == w["allocs"], g["it"]
        assert g["edges"] == w["edges"], g["it"]
        assert g["admitted"] == w["admitted"], g["it"]
    assert dc.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(dc.coverage_map())) == ref["coverage"]
    assert [_digest(e[0]) for e in dc.host_entries] == ref["corpus"]
    dc.close()


@pytest.mark.parametrize("name", ["amax", "amin", "rotm", "dot"])
def test_pipelined_rounds_equal_sequential(engine_cls, name):
    """Speculative round pipelining (depth 4) reproduces the reference's batched
    records exactly, including rounds that admit children (re-submission path)."""
    data = golden("ref_batched.json")
    cfg = data["config"]
    ref = data["runs"][name]
    m = bench_manifest(name)
    dc = engine_cls(m, master_seed=cfg["master_seed"])
    got = []
    dc.run_rounds(1, cfg["iterations"] + 1, cfg["round_size"], depth=4,
                  on_round=lambda res: got.extend(dc.round_records(res)))
    assert len(got) == len(ref["records"])
    for g, w in zip(got, ref["records"]):
        assert _digest(g["child"]) == w["child"], g["it"]
        assert g["report"] == w["report"], g["it"]
        assert g["edges"] == w["edges"], g["it"]
        assert g["admitted"] == w["admitted"], g["it"]
    assert dc.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(dc.coverage_map())) == ref["coverage"]
    assert [_digest(e[0]) for e in dc.host_entries] == ref["corpus"]
    dc.close()


def test_fuzz_loop_api_matches_batched_reference(engine_cls, tmp_path):
    """The reference-shaped fuzz_loop (public API) over the same contract."""
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    data = golden("ref_batched.json")
    cfg = data["config"]
    ref = data["runs"]["amax"]
    m = bench_manifest("amax")
    s = fuzz_loop(m, CampaignConfig(master_seed=cfg["master_seed"], iterations=cfg["iterations"],
                                    round_size=cfg["round_size"], pipeline_depth=3, out_dir=tmp_path / "out"))
    assert s.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(s.coverage)) == ref["coverage"]
    assert [_digest(e.tc) for e in s.corpus.entries] == ref["corpus"]
    assert s.compute_runs == cfg["iterations"]
    assert (tmp_path / "out" / "findings.txt").read_text() == ref["findings"]
    crashes = sorted(p.name for p in (tmp_path / "out" / "crashes").iterdir())
    assert len(crashes) == len(s.findings)


def test_pipelined_equals_sequential_under_overlap(engine_cls):
    """Rounds of the matmul target run long enough to overlap on the device; the
    pipelined campaign must equal the one-round-at-a-time campaign bit for bit."""
    import numpy as np
    from conftest import workload_manifest
    from paper_2603_05725_b200.lowering import VERDICT
    m = workload_manifest("matmul")

    def campaign(depth):
        dc = engine_cls(m, master_seed=3)
        digests = []

        def keep(res):
            v = res.slot.verdicts[:res.executed * VERDICT.itemsize].cpu().numpy().view(VERDICT).copy()
            v["where"] = 0   # diagnostics (SM id, ns spent): not part of the result
            e = res.slot.ecnt[:res.executed * max(dc.E, 1)].cpu().numpy()
            digests.append(hashlib.sha256(v.tobytes() + e.tobytes()).hexdigest())

        if depth == 1:
            for k in range(6):
                keep(dc.run_round(1 + k * 4096, 4096))
        else:
            dc.run_rounds(1, 1 + 6 * 4096, 4096, depth=depth, on_round=keep)
        out = (digests, dc.findings.render_text(), report_to_rec(build_report(dc.coverage_map())),
               [e[0].id for e in dc.host_entries])
        dc.close()
        return out

    seq = campaign(1)
    pip = campaign(6)
    assert seq[0] == pip[0]
    assert seq[1:] == pip[1:]


@pytest.mark.parametrize("stem", ["matmul", "vadd", "ctxchain", "structcfg"])
@pytest.mark.parametrize("depth,soft_cap", [(1, None), (3, None), (3, 0), (2, 300)])
def test_workloads_match_reference(engine_cls, stem, depth, soft_cap):
    """C1 (vadd, off-by-one OOB write), C2 (matmul, stride/size OOB), C3 (3-launch
    chain, OOB + use-after-free) and C4 (struct argument, 200-seed corpus, fixed
    fan-out 8) on the device vs the reference's batched records
    (tests/golden/ref_workloads.json).  soft_cap: long inputs deferred to the tail
    pass (None = default, 0 = off, 300 = most inputs deferred) -- the results must
    not depend on it."""
    from conftest import workload_case
    ref = golden("ref_workloads.json")[stem]
    m, kw, R, iters = workload_case(stem)
    dc = engine_cls(m, master_seed=11, soft_cap=soft_cap, **kw)
    got = []
    dc.run_rounds(1, iters + 1, R, depth=depth, on_round=lambda res: got.extend(dc.round_records(res)))
    assert len(got) == len(ref["records"])
    for g, w in zip(got, ref["records"]):
        assert g["parent"] == w["parent"], g["it"]
        assert _digest(g["child"]) == w["child"], g["it"]
        assert g["status"] == w["status"], g["it"]
        assert g["report"] == w["report"], g["it"]
        assert g["retired"] == w["retired"], g["it"]
        assert g["allocs"] == w["allocs"], g["it"]
        assert g["edges"] == w["edges"], g["it"]
        assert g["admitted"] == w["admitted"], g["it"]
    assert dc.findings.render_text() == ref["findings"]
    assert report_to_rec(build_report(dc.coverage_map())) == ref["coverage"]
    assert [_digest(e[0]) for e in dc.host_entries] == ref["corpus"]
    dc.close()


def test_context_sensitive_map(engine_cls):
    """C3: the 16 MiB context-sensitive hashed map (derived view) equals the map
    recomputed from the reference's per-input edge counts."""
    from conftest import workload_manifest
    from paper_2603_05725_b200.lowering import ctx_edge_hashes, ctx_slot
    ref = golden("ref_workloads.json")["ctxchain"]
    m = workload_manifest("ctxchain")
    dc = engine_cls(m, master_seed=11, ctx_map_bits=24)
    dc.run_rounds(1, 301, 100, depth=2)
    hashes = ctx_edge_hashes(dc.low, m)
    index = {(name, tuple(e)): j for j, (name, e) in enumerate(dc.low.edge_names)}
    want = sorted({ctx_slot(hashes[index[(k, (a, b))]], c, 24)
                   for r in ref["records"] for k, es in r["edges"].items() for a, b, c in es})
    assert dc.ctx_map_slots().tolist() == want
    assert int(dc.ctx_new.item()) == len(want)
    assert report_to_rec(build_report(dc.coverage_map())) == ref["coverage"]
    dc.close()


def test_struct_corpus_full_size_prefix(engine_cls):
    """C4 at full size: a 10,000-seed corpus (sample_valid_testcase), 64 children
    per seed, one round of 640,000 inputs on the device; the first 256 inputs
    (records are prefix-consistent within a round) equal the CPU oracle's."""
    from conftest import workload_manifest
    from oracle.loop import batched_loop
    from paper_2603_05725_b200.testcase import Stream, sample_valid_testcase
    m = workload_manifest("structcfg")
    seeds = tuple(sample_valid_testcase(m.argspecs, Stream(11, (7 << 40) + k)) for k in range(9999))
    R = 10_000 * 64
    dc = engine_cls(m, master_seed=11, extra_seeds=seeds, fanout=64)
    res = dc.run_round(1, R)
    assert res.executed == R
    got = dc.round_records(res)[:256]
    ref = batched_loop(m, master_seed=11, iterations=256, round_size=R, extra_seeds=seeds, fanout=64).records
    for g, w in zip(got, ref):
        assert g["parent"] == w["parent"], g["it"]
        assert g["child"].id == w["child"].id, g["it"]
        assert g["report"] == w["report"], g["it"]
        assert g["retired"] == w["retired"], g["it"]
        assert g["edges"] == w["edges"], g["it"]
        assert g["admitted"] == w["admitted"], g["it"]
    dc.close()


@pytest.mark.parametrize("name", bench_names())
def test_group_parallel_bulk_matches_reference(engine_cls, name, monkeypatch):
    """Every input through the group-parallel mode (simulated threads of a launch on
    the lanes of a group, conflict tags, in-place sequential re-run of conflicting
    chunks, WAW acceptance when memory is dead): the bundled harnesses include
    cross-thread read-modify-writes (amax/amin/asum/nrm2/dot reduce into out[0]),
    so conflicts, re-runs and WAW all occur.  Records equal the reference's."""
    monkeypatch.setenv("SFG_BULK_GROUP", "32")  # capped to the program's group size per launch
    data = golden("ref_batched.json")
    cfg = data["config"]
    ref = data["runs"][name]
    m = bench_manifest(name)
    dc = engine_cls(m, master_seed=cfg["master_seed"], soft_cap=200)
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
    dc.close()


def test_order_mask_is_control_taint(engine_cls):
    """sfg_order groups inputs by the arguments that can steer control flow: for the
    matmul target the loop bounds m, n, k and, through the sanitizer's verdicts on
    the addresses they form, a, b, c and the leading dimensions; structcfg's f32
    alpha is pure data."""
    from conftest import workload_manifest
    dc = engine_cls(workload_manifest("matmul"), master_seed=11)
    names = [s.name for s in dc.specs]
    mask = dc.L.sfg_program_order_mask(dc.h)
    assert {names[a] for a in range(len(names)) if mask >> a & 1} == set(names)
    dc.close()
    dc = engine_cls(workload_manifest("structcfg"), master_seed=11)
    names = [s.name for s in dc.specs]
    mask = dc.L.sfg_program_order_mask(dc.h)
    assert {names[a] for a in range(len(names)) if mask >> a & 1} == {"cfg", "x", "y"}
    dc.close()


def _trace_text(events):
    import io
    from paper_2603_05725_b200.hooks import TraceHooks, dispatch
    buf = io.StringIO()
    dispatch(TraceHooks(buf), events)
    return buf.getvalue()


@pytest.mark.parametrize("name", bench_names())
def test_trace_events_match_reference(engine_cls, name):
    """Device trace mode (sfg_execute_trace) reproduces the reference's TraceHooks
    stream (executor.py:122-135) line for line on sampled inputs."""
    ref = golden("ref_traces.json")["inputs"][name]
    m = bench_manifest(name)
    dc = engine_cls(m, master_seed=1)
    tcs = [parse_testcase(r["testcase"])[0] for r in ref]
    outs = dc.execute_testcases(tcs, iteration0=1, trace=True)
    for out, r in zip(outs, ref):
        text = _trace_text(out["events"])
        assert text.splitlines()[:len(r["head"])] == r["head"]
        assert len(text.splitlines()) == r["n_lines"]
        assert hashlib.sha256(text.encode()).hexdigest() == r["sha256"]
    dc.close()


@pytest.mark.parametrize("name", ["dot", "amax"])
def test_traced_campaign_matches_reference(engine_cls, name):
    """fuzz_loop(hooks=TraceHooks) over the batched-round contract: the whole event
    stream of the campaign equals the reference functions' (make_golden traces)."""
    import io
    from paper_2603_05725_b200.campaign import CampaignConfig, TraceHooks, fuzz_loop
    data = golden("ref_traces.json")
    cfg, ref = data["campaign_config"], data["campaigns"][name]
    buf = io.StringIO()
    fuzz_loop(bench_manifest(name), CampaignConfig(master_seed=cfg["master_seed"], iterations=cfg["iterations"],
                                                   round_size=cfg["round_size"], hooks=TraceHooks(buf)))
    text = buf.getvalue()
    assert len(text.splitlines()) == ref["n_lines"]
    assert text.splitlines()[:len(ref["head"])] == ref["head"]
    assert hashlib.sha256(text.encode()).hexdigest() == ref["sha256"]


@pytest.mark.parametrize("case", ["init_overflow", "compute_out_of_space"])
def test_fatal_conditions_raise_reference_exceptions(engine_cls, case):
    """fuzz_loop raises the reference's exception class (and message) for a failing
    INIT phase (CampaignFatalError) and for a COMPUTE allocation that does not fit
    (OutOfSpaceError), tests/golden/ref_errors.json (made by the reference)."""
    from paper_2603_05725_b200.baseline import MemConfig
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    from paper_2603_05725_b200.manifest import harness_from_text
    data = golden("ref_errors.json")
    c = data["cases"][case]
    m = harness_from_text(c["harness"], data["kernel"], f"{case}/harness.man")
    with pytest.raises(Exception) as ei:
        fuzz_loop(m, CampaignConfig(master_seed=11, iterations=8, mem_config=MemConfig(**c["mem"])))
    assert type(ei.value).__name__ == c["raises"]
    assert str(ei.value) == c["message"]


@pytest.mark.parametrize("key", sorted(golden("ref_fuzzloop.json")))
@pytest.mark.parametrize("round_size", [64, 4096])
def test_sequential_fuzz_loop_matches_reference_output_dir(engine_cls, key, round_size, tmp_path):
    """discipline="sequential": the reference fuzz_loop's own semantics (one worker
    stream, live corpus; rounds generated in order on the device and cut after each
    admission).  The output directory equals the reference fuzz_loop's
    (tests/golden/ref_fuzzloop.json, made by the reference): findings.txt,
    coverage.rec / coverage.txt, corpus and crash file names (sha256 test-case ids),
    summary.rec -- whatever the round size."""
    from paper_2603_05725_b200.campaign import CampaignConfig, fuzz_loop
    name, seed, iters = key.split("/")
    want = golden("ref_fuzzloop.json")[key]
    d = tmp_path / "out"
    s = fuzz_loop(bench_manifest(name), CampaignConfig(master_seed=int(seed), iterations=int(iters), out_dir=d,
                                                       discipline="sequential", round_size=round_size,
                                                       **want["kw"]))
    assert (d / "findings.txt").read_text() == want["findings"]
    assert (d / "coverage.rec").read_text() == want["coverage_rec"]
    assert (d / "coverage.txt").read_text() == want["coverage_txt"]
    assert sorted(p.name for p in (d / "corpus").iterdir()) == want["corpus"]
    assert sorted(p.name for p in (d / "crashes").iterdir()) == want["crashes"]
    assert s.to_rec() == want["summary"]


WIDE_SIR = """\
# pointer registers beyond int64: a 64-bit load into a pointer register and a
# near-2^63 immediate plus i32 offsets (the 128-bit register form of the
# specialized kernel; addresses in reports must stay exact)
kernel widereg(x:ptr.global, n:i32, k:i32) regs=8
  ld.global.b64 %a1, [%a0]
  setp.lt %p0, %r0, 4
  bra %p0, small
  mov %a2, 9223372036854775792
  add %a2, %a2, %r0
  add %a2, %a2, %r1
  ld.global.b32 %r2, [%a2]
  exit
small:
  add %a1, %a1, %r1
  ld.global.b32 %r3, [%a1]
  mov %a3, %a0
  add %a3, %a3, %r0
  st.global.b32 [%a3], %r1
  exit
"""

WIDE_MAN = """\
program widereg.sir

argspec x ptr global i32 count=4 seed=seq lo=-4 hi=4
argspec n i32 seed=0 lo=0 hi=8
argspec k i32 seed=0 lo=-8 hi=8

init:
  alloc ws global 4096
  copy_in ws zeros:4096
compute:
  launch widereg grid=1 block=2 args=arg:0,arg:1,arg:2
term:
  free ws
"""


def test_wide_pointer_registers_match_oracle(engine_cls):
    """A kernel whose pointer registers leave int64 (a 64-bit load into one, a
    near-2^63 immediate plus offsets) keeps the specialized kernel's 128-bit
    register form; every input of a batched campaign equals the CPU oracle:
    child, verdict line (exact wild addresses), retired count, edges, admission."""
    from oracle.loop import batched_loop
    from paper_2603_05725_b200.manifest import harness_from_text
    m = harness_from_text(WIDE_MAN, WIDE_SIR, "widereg/harness.man")
    n, R = 1024, 256
    want = batched_loop(m, master_seed=5, iterations=n, round_size=R).records
    dc = engine_cls(m, master_seed=5)
    import ctypes
    nb = dc.L.sfg_program_jit_source(dc.h, None, 0)
    buf = ctypes.create_string_buffer(nb + 1)
    dc.L.sfg_program_jit_source(dc.h, buf, nb + 1)
    assert "i128 a1 =" in buf.value.decode()   # the 128-bit register form was generated
    got = []
    dc.run_rounds(1, n + 1, R, depth=2, on_round=lambda res: got.extend(dc.round_records(res)))
    assert len(got) == len(want)
    kinds = set()
    for g, w in zip(got, want):
        assert _digest(g["child"]) == _digest(w["child"]), g["it"]
        assert (g["status"], g["report"], g["retired"]) == (w["status"], w["report"], w["retired"]), g["it"]
        assert (g["edges"], g["admitted"], g["allocs"]) == (w["edges"], w["admitted"], w["allocs"]), g["it"]
        if w["report"]:
            f = dict(t.split("=", 1) for t in w["report"].split()[1:] if "=" in t)
            a = f["addr"][2:]
            a = -int(a[1:], 16) if a.startswith("-") else int(a, 16)
            kinds.add((f["class"], f["iid"], a >= 1 << 63, a < 0))
    # wild addresses past 2^63 and below 0, out-of-bounds and space mismatches
    assert len(kinds) >= 5 and any(k[2] for k in kinds) and any(k[3] for k in kinds)
    dc.close()


@pytest.mark.parametrize("name", ["matmul", "vadd", "structcfg", "dot", "amax", "rotm", "axpy"])
def test_seqgen_equals_one_thread_walk(engine_cls, name):
    """The sequential discipline's parallel generator (seqgen: every candidate child
    boundary of the worker stream draws one child, pointer doubling finds the
    boundaries reachable from the worker state, children generated in parallel)
    gives the one-thread walk's children, values, int picks and stream states bit
    for bit over 20,000 children -- the walk is the path pinned to the reference
    fuzz_loop (test_sequential_fuzz_loop_matches_reference_output_dir)."""
    from conftest import workload_manifest
    from paper_2603_05725_b200.engine import CHILD
    m = bench_manifest(name) if name in bench_names() else workload_manifest(name)
    dc = engine_cls(m, master_seed=11, sequential=True)
    dc.new_worker(0)
    dc.run_rounds(1, 1 + 512, 512)            # one-thread rounds until the rotation counts saturate
    assert dc._counts_sat
    # no corpus entry may leave the recent window inside the generated range
    window = int(dc.low.prog["window"])
    it0 = max([513] + [adm + window + 1 for _, adm, seed in dc.host_entries if not seed])
    n = 20000
    a = dc.seq_generate(it0, n, parallel=False)
    b = dc.seq_generate(it0, n, parallel=True)
    found = int(b[4][0])
    assert found == n, (found, dc.seq_truncations)
    assert (a[0] == b[0]).all()
    assert (a[1] == b[1]).all()
    assert (a[2] == b[2]).all()
    assert (_stream_states(a[3]) == _stream_states(b[3])).all()
    # a candidate range too short for the round truncates it exactly: the children
    # found are the walk's, and the resume state after them is exact
    c = dc.seq_generate(it0, n, parallel=True, words=3000)
    k = int(c[4][0])
    assert 0 < k < n
    cw, sb = CHILD.itemsize, dc.state_bytes
    assert (c[0][:k * cw] == a[0][:k * cw]).all()
    assert (_stream_states(c[3][:(k + 1) * sb]) == _stream_states(a[3][:(k + 1) * sb])).all()
    dc.close()


def _stream_states(raw):
    """SfgStream records (philox.cuh) with the bytes that carry no state cleared: the
    32-bit cache word when no half-word is cached, and the padding."""
    import numpy as np
    st = np.frombuffer(raw.tobytes(), dtype=np.dtype([("ctr", "<u8", (4,)), ("key", "<u8", (2,)), ("buf", "<u8", (4,)),
                                                      ("pos", "<u4"), ("has32", "<u4"), ("cache32", "<u4"),
                                                      ("pad", "<u4")])).copy()
    assert st.dtype.itemsize == 96
    st["cache32"][st["has32"] == 0] = 0
    st["pad"] = 0
    return st


@pytest.mark.parametrize("name", ["matmul", "structcfg", "dot", "rotm"])
def test_duplicate_inputs_run_once(engine_cls, name, monkeypatch):
    """sfg_dedupe: children with the same parent and the same set of ops run once
    and their duplicates take the verdict and edge row; every per-input record of
    a batched campaign equals the one where every input runs (SFG_DEDUPE=0), and
    a large share of a round are duplicates."""
    from conftest import workload_manifest
    m = bench_manifest(name) if name in bench_names() else workload_manifest(name)
    runs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SFG_DEDUPE", flag)
        dc = engine_cls(m, master_seed=5)
        got = []
        dc.run_rounds(1, 1 + 3 * 65536, 65536, depth=3, on_round=lambda res: got.extend(dc.round_records(res)))
        if flag == "1":
            S = dc.slots[0]
            rep = S.rep[:S.n].cpu().numpy()
            runs["dups"] = int((rep != np.arange(S.n)).sum())
        runs[flag] = (got, dc.findings.render_text(), report_to_rec(build_report(dc.coverage_map())))
        dc.close()
    a, b = runs["1"], runs["0"]
    assert a[1] == b[1] and a[2] == b[2] and len(a[0]) == len(b[0])
    for x, y in zip(a[0], b[0]):
        assert _digest(x["child"]) == _digest(y["child"])
        assert (x["status"], x["report"], x["retired"], x["allocs"], x["edges"], x["admitted"]) == \
               (y["status"], y["report"], y["retired"], y["allocs"], y["edges"], y["admitted"]), x["it"]
    assert runs["dups"] > 1000
