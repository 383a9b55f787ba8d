"""Generate golden fixtures by running the REAL reference (simt_forge) here.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes (all small, committed):
  bench_assets.json   the 11 bundled benchmark programs/harnesses, their 44
                      seeded-bug variants and trigger traces (workload definitions)
  ref_variants.json   execute_once verdict line for every trigger variant
  ref_sampled.json    valid-domain + special-value inputs with diff readbacks
  ref_batched.json    per-input records of the batched-round contract driven by
                      the reference's own functions (schedule_next, mutate_testcase
                      with a shared MutationSchedule, PhaseRunner, _absorb order)
  ref_fuzzloop.json   reference fuzz_loop campaign outputs (findings, coverage,
                      summary, corpus) for a few configs
  ref_workloads.json  the same batched records for this repo's synthetic
                      workloads (paper_2603_05725_b200/workloads)
  ref_errors.json     the exception class the reference fuzz_loop raises for
                      failing harnesses (INIT failure, out of space)
  ref_nests.json      matmul loop nests with loads/stores to the budget, to the
                      row exit, and with failing nest guards (records per budget)
  ref_traces.json     ExecHooks event streams (TraceHooks "EV mem" / "EV cf"
                      lines): per sampled input of every benchmark, and for a
                      traced batched campaign (dot, amax)
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

from simt_forge import bench as rb  # noqa: E402
from simt_forge import campaign as rc  # noqa: E402
from simt_forge.coverage import CoverageMap, build_report, new_edges_since, report_to_rec  # noqa: E402
from simt_forge.device_memory import DeviceMemoryImage  # noqa: E402
from simt_forge.mutation import (ArrayValue, FloatValue, IntValue, MutationSchedule,  # noqa: E402
                                 TestCase, apply_trace, mutate_testcase,
                                 sample_valid_testcase, serialize_testcase)
from simt_forge.rng import Stream  # noqa: E402

KEYBASE = 1 << 32


def digest(tc) -> str:
    return hashlib.sha256(serialize_testcase(tc, with_id=False).encode()).hexdigest()[:32]


def edges_json(delta):
    return {k: sorted([list(e) + [c] for e, c in v.items()]) for k, v in delta.edge_counts.items() if v}


def assets():
    out = {}
    for b in rb.list_benchmarks():
        ent = {"kernel": (b.root / "kernel.sir").read_text(),
               "harness": (b.root / "harness.man").read_text(), "variants": {}}
        for v in b.variants():
            vd = {"trigger": v.trigger_path.read_text()}
            if (v.root / "harness.man").exists():
                vd["harness"] = (v.root / "harness.man").read_text()
                vd["kernel"] = (v.root / "kernel.sir").read_text()
            ent["variants"][v.bug_class] = vd
        out[b.name] = ent
    return out


def variants():
    out = {}
    for b in rb.list_benchmarks():
        for v in b.variants():
            expected, ops = rb.load_trigger(v)
            m = rc.load_harness(v.harness_path)
            tc = rb.build_trigger_testcase(m, ops)
            cov = CoverageMap.for_program(m.program)
            res, _ = rc.execute_once(m, tc, coverage=cov)
            out[f"{b.name}/{v.bug_class}"] = {
                "expected": expected, "status": res.status, "retired": res.retired,
                "report": res.report.to_line() if res.report else None, "edges": edges_json(cov)}
    return out


SPECIAL_F32 = [0x7FA00000, 0xFFC12345, 0x7F800000, 0xFF800000, 0x00000001, 0x80000000,
               0x7F7FFFFF, 0x3E99999A, 0x4B800001, 0xCF000000, 0x4F000000, 0x7FFFFFFF]


def sampled():
    """Valid-domain inputs plus special-value arrays; readbacks pin f32/i32 bits."""
    out = {}
    for bi, b in enumerate(rb.list_benchmarks()):
        m = b.load()
        image = DeviceMemoryImage()
        runner = rc.PhaseRunner(m, image, diff_readback=True)
        runner.run_phase(rc.INIT, m.seed(1), iteration=0)
        runner.mark_baseline()
        snap = image.snapshot()
        rng = Stream(99, bi)
        recs = []
        for i in range(24):
            tc = sample_valid_testcase(m.argspecs, rng)
            if i >= 12:  # sprinkle special bit patterns into float arrays/scalars
                args = list(tc.args)
                for k, v in enumerate(args):
                    if isinstance(v, ArrayValue) and v.elem == "f32" and v.data:
                        words = list(struct.unpack(f"<{len(v.data) // 4}I", v.data))
                        for j in range(0, len(words), 3):
                            words[j] = SPECIAL_F32[(i + j) % len(SPECIAL_F32)]
                        args[k] = ArrayValue(struct.pack(f"<{len(words)}I", *words), v.elem,
                                             v.extents, v.space)
                    elif isinstance(v, FloatValue):
                        args[k] = FloatValue(SPECIAL_F32[(i + k) % len(SPECIAL_F32)])
                tc = TestCase(tuple(args), tc.rng_seed)
            image.restore(snap)
            runner.reset_to_baseline()
            cov = CoverageMap.for_program(m.program)
            res = runner.run_phase(rc.COMPUTE, tc, coverage=cov, iteration=i + 1)
            recs.append({"testcase": serialize_testcase(tc, with_id=False), "status": res.status,
                         "retired": res.retired,
                         "report": res.report.to_line() if res.report else None,
                         "readouts": {k: v.hex() for k, v in res.readouts.items()},
                         "edges": edges_json(cov)})
        out[b.name] = recs
    return out


def batched(m, *, master_seed, iterations, round_size, stop_bug_class=None,
            stop_on_first_finding=False, extra_seeds=(), fanout=0, hooks=None, budget=1_000_000):
    """Batched-round contract on the reference's own functions.  fanout > 0: input
    it mutates round-corpus entry ((it - 1) // fanout) % len (no scheduling draw)."""
    specs = m.argspecs
    seed_tc = m.seed(master_seed)
    corpus = rc.Corpus()
    corpus.add_seed(seed_tc)
    for tc in extra_seeds:
        corpus.add_seed(tc)
    findings = rc.FindingsLog()
    gcov = CoverageMap.for_program(m.program)
    sched = MutationSchedule()
    image = DeviceMemoryImage(rng=Stream(master_seed, 2000))
    runner = rc.PhaseRunner(m, image, hooks=hooks, instruction_budget=budget)
    assert runner.run_phase(rc.INIT, seed_tc, iteration=0).status == "ok"
    runner.mark_baseline()
    snap = image.snapshot()
    recs = []
    round_corpus = None
    stop = "iterations"
    want = stop_bug_class
    for it in range(1, iterations + 1):
        if (it - 1) % round_size == 0:
            round_corpus = rc.Corpus(list(corpus.entries))
        image.restore(snap)
        runner.reset_to_baseline()
        if it == 1:
            child, pidx = seed_tc, -1
        else:
            s = Stream(master_seed, KEYBASE + it)
            if fanout:
                pidx = ((it - 1) // fanout) % len(round_corpus.entries)
                parent = round_corpus.entries[pidx].tc
            else:
                parent = rc.schedule_next(round_corpus, s, it)
                pidx = next(i for i, e in enumerate(round_corpus.entries) if e.tc is parent)
            child = mutate_testcase(parent, specs, sched, s)
        delta = gcov.fresh()
        first = image._next_alloc_id
        out = runner.run_phase(rc.COMPUTE, child, coverage=delta, iteration=it)
        fresh = new_edges_since(delta, gcov)
        gcov.merge_from(delta)
        rec = {"it": it, "parent": pidx, "child": digest(child), "rng_seed": str(child.rng_seed),
               "trace": [op.encode() for op in child.trace], "status": out.status,
               "retired": out.retired, "allocs": image._next_alloc_id - first,
               "edges": edges_json(delta), "admitted": False, "report": None}
        halt = None
        if out.report is not None:
            out.report.iteration = it
            rec["report"] = out.report.to_line()
            findings.add(out.report)
            if stop_on_first_finding:
                halt = "first_finding"
            elif want is not None and out.report.bug_class.value == want:
                halt = f"bug_class:{want}"
        elif fresh and it != 1:
            corpus.admit(child, it)
            rec["admitted"] = True
        recs.append(rec)
        if halt:
            stop = halt
            break
    return {"records": recs, "findings": findings.render_text(),
            "coverage": report_to_rec(build_report(gcov)),
            "global_edges": edges_json(gcov), "stop": stop,
            "corpus": [digest(e.tc) for e in corpus.entries]}


BATCH_CFG = dict(master_seed=11, iterations=600, round_size=128)


def batched_all():
    return {b.name: batched(b.load(), **BATCH_CFG) for b in rb.list_benchmarks()}


def fuzzloops(tmp):
    out = {}
    for name, seed, iters, kw in (("dot", 11, 400, {}), ("amax", 7, 300, {}),
                                  ("rotm", 5, 300, {}),
                                  ("axpy", 11, 3000, {"stop_bug_class": "SPATIAL_OOB"})):
        m = rb.get_benchmark(name).load()
        d = Path(tmp) / f"{name}-{seed}"
        s = rc.fuzz_loop(m, rc.CampaignConfig(master_seed=seed, iterations=iters, out_dir=d, **kw))
        out[f"{name}/{seed}/{iters}"] = {
            "kw": kw, "summary": s.to_rec(), "findings": (d / "findings.txt").read_text(),
            "coverage_rec": (d / "coverage.rec").read_text(),
            "coverage_txt": (d / "coverage.txt").read_text(),
            "corpus": sorted(p.name for p in (d / "corpus").iterdir()),
            "crashes": sorted(p.name for p in (d / "crashes").iterdir()),
        }
    return out


STRUCT_SEEDS = 199          # + the manifest seed = 200 corpus entries
STRUCT_SEED_KEY = 7 << 40   # sample_valid_testcase(specs, Stream(11, STRUCT_SEED_KEY + k))


def struct_seeds(m, n=STRUCT_SEEDS, master_seed=11):
    return [sample_valid_testcase(m.argspecs, Stream(master_seed, STRUCT_SEED_KEY + k)) for k in range(n)]


def workloads():
    wdir = REPO / "paper_2603_05725_b200" / "workloads"
    out = {}
    for man in sorted(wdir.glob("*.man")):
        m = rc.load_harness(man)
        if man.stem == "structcfg":   # C4: seed corpus + 8 children per seed, two rounds
            seeds = struct_seeds(m)
            out[man.stem] = batched(m, master_seed=11, iterations=3200, round_size=1600,
                                    extra_seeds=seeds, fanout=8)
            out[man.stem]["seeds"] = [serialize_testcase(t) for t in seeds]
        else:
            out[man.stem] = batched(m, master_seed=11, iterations=300, round_size=100)
    return out


TRACE_INPUTS = (0, 1, 2, 12)
TRACE_CAMPAIGN = dict(master_seed=11, iterations=48, round_size=16)


def _trace_summary(text: str, head: int = 24) -> dict:
    lines = text.splitlines()
    return {"n_lines": len(lines), "sha256": hashlib.sha256(text.encode()).hexdigest(), "head": lines[:head]}


def traces():
    """Event streams of the reference's TraceHooks (executor.py:122-135)."""
    import io
    from simt_forge.executor import TraceHooks
    from simt_forge.mutation import parse_testcase
    samp = json.loads((HERE / "ref_sampled.json").read_text())
    out = {"inputs": {}, "campaigns": {}, "campaign_config": TRACE_CAMPAIGN}
    for b in rb.list_benchmarks():
        m = b.load()
        recs = []
        for i in TRACE_INPUTS:
            tc, _ = parse_testcase(samp[b.name][i]["testcase"], m.argspecs)
            buf = io.StringIO()
            image = DeviceMemoryImage()
            runner = rc.PhaseRunner(m, image, hooks=TraceHooks(buf))
            runner.run_phase(rc.INIT, m.seed(1), iteration=0)
            buf.seek(0)
            buf.truncate()
            runner.run_phase(rc.COMPUTE, tc, iteration=i + 1)
            recs.append({"testcase": samp[b.name][i]["testcase"], **_trace_summary(buf.getvalue())})
        out["inputs"][b.name] = recs
    for name in ("dot", "amax"):
        m = next(b for b in rb.list_benchmarks() if b.name == name).load()
        buf = io.StringIO()
        batched(m, hooks=TraceHooks(buf), **TRACE_CAMPAIGN)
        out["campaigns"][name] = _trace_summary(buf.getvalue())
    return out


# Error behaviour (campaign.py:79-80, 685-688, 723-725; device_memory.py:62-63,
# 426-430): which exception the reference's fuzz_loop raises, for harnesses
# written here in the reference's own formats.
ERROR_KERNEL = """\
kernel poke(buf:ptr.global, n:i32) regs=8
  st.global.b32 [%a0], %r0
  exit
"""
ERROR_CASES = {
    # INIT copies 128 bytes into a 64-byte buffer: the init phase fails on the seed
    "init_overflow": ("argspec b ptr global i32 count=4 seed=zeros lo=0 hi=9\n"
                      "argspec n i32 seed=3 lo=0 hi=9\n\n"
                      "init:\n  alloc scratch global 64\n  copy_in scratch hex:" + "00" * 128 + "\n"
                      "compute:\n  launch poke grid=1 block=1 args=arg:0,arg:1\n"
                      "term:\n  free scratch\n", {}),
    # a COMPUTE allocation larger than the global space
    "compute_out_of_space": ("argspec b ptr global i32 count=4 seed=zeros lo=0 hi=9\n"
                             "argspec n i32 seed=3 lo=0 hi=9\n\n"
                             "compute:\n  alloc big global 100000\n"
                             "  launch poke grid=1 block=1 args=arg:0,arg:1\n  free big\n",
                             {"global_size": 65536}),
}


def errors(tmp):
    from simt_forge.device_memory import MemConfig
    out = {}
    for name, (body, mem) in ERROR_CASES.items():
        d = Path(tmp) / name
        d.mkdir()
        (d / "kernel.sir").write_text(ERROR_KERNEL)
        (d / "harness.man").write_text("program kernel.sir\n\n" + body)
        m = rc.load_harness(d / "harness.man")
        try:
            rc.fuzz_loop(m, rc.CampaignConfig(master_seed=11, iterations=8, mem_config=MemConfig(**mem)))
            out[name] = {"raises": None}
        except Exception as e:  # noqa: BLE001 - the class is the golden value
            out[name] = {"raises": type(e).__name__, "message": str(e)}
    return {"kernel": ERROR_KERNEL, "cases": {k: {"harness": "program kernel.sir\n\n" + v[0], "mem": v[1],
                                                 **out[k]} for k, v in ERROR_CASES.items()}}


# Long pure-register loops (the JIT's loop summaries, csrc/jit.cu analyse_cycle):
# exits by == / != / <= / > compares of wrapping i32 induction variables, and
# budget exhaustion at every position of the loop body (budgets 10^6 + k).
LOOP_SIR = """\
kernel spin(out:ptr.global, x:i32, step:i32, lim:i32, stop:i32) regs=8
  mov %r5, 0
top:
  setp.eq %p1, %r0, %r3
  bra %p1, hit
  add %r0, %r0, %r1
  sub %r5, %r5, -1
  setp.gt %p0, %r5, %r2
  bra %p0, fin
  bra top
hit:
  st.global.b32 [%a0], %r5
  exit
fin:
  st.global.b32 [%a0+4], %r0
  exit

kernel spin2(out:ptr.global, x:i32, step:i32, lim:i32, stop:i32) regs=8
  mov %r6, 7
again:
  add %r0, %r0, %r1
  setp.ne %p2, %r0, %r3
  bra !%p2, found
  mov %r6, 9
  setp.le %p3, %r0, %r2
  bra !%p3, again
  st.global.b32 [%a0+8], %r6
  exit
found:
  st.global.b32 [%a0+12], %r0
  exit
"""


def loop_manifest(kernel: str) -> str:
    return ("program loops.sir\n\n"
            "argspec out ptr global i32 count=4 seed=zeros lo=0 hi=9\n"
            "argspec x i32 seed=0 lo=-100 hi=100\n"
            "argspec step i32 seed=8 lo=-9 hi=9\n"
            "argspec lim i32 seed=400 lo=0 hi=1000\n"
            "argspec stop i32 seed=4000 lo=0 hi=1000\n\n"
            "compute:\n"
            f"  launch {kernel} grid=1 block=2 args=arg:0,arg:1,arg:2,arg:3,arg:4\n"
            "  copy_out arg:0\n")


M31 = (1 << 31) - 1
LOOP_INPUTS = {
    # (x, step, lim, stop)
    "spin": [(0, 8, 10 ** 9, 8 * 50000), (5, 0x10000001, 10 ** 9, (5 + 1000 * 0x10000001) & 0xFFFFFFFF),
             (0, 3, 200000, 1), (0, 0, M31, 1), (-(1 << 31) + 100, -7, 10 ** 9, 2000000),
             (7, 1, 30000, 30007 + 1), (0, -1, 10 ** 6, -123457)],
    "spin2": [(M31, -1, M31 - 100000, -5), (M31, -1, M31 - 300000, -5), (100, 1, 50, -7),
              (100, 0x7FFFFFFF, 50, 3), (0, 4, -100, 400000), (-5, 3, -10, 2 ** 31 - 2)],
}
LOOP_BUDGETS = [10 ** 6 + k for k in range(7)] + [200003]
MATMUL_LOOPS = [(M31, 0), (M31, -8), (400000, 0), (M31, -(1 << 31))]   # (m, n)
LOOP_CAMPAIGN = dict(master_seed=7, iterations=2048, round_size=512, budget=50000)


def loops():
    from simt_forge.mutation import IntValue
    import tempfile
    out = {"kernel": LOOP_SIR, "manifests": {}, "inputs": {}, "campaigns": {}, "campaign_config": LOOP_CAMPAIGN,
           "budgets": LOOP_BUDGETS}
    with tempfile.TemporaryDirectory() as tmp:
        (Path(tmp) / "loops.sir").write_text(LOOP_SIR)
        cases = []
        for kern in ("spin", "spin2"):
            man = loop_manifest(kern)
            out["manifests"][kern] = man
            (Path(tmp) / f"{kern}.man").write_text(man)
            m = rc.load_harness(Path(tmp) / f"{kern}.man")
            seed = m.seed(1)
            for vals in LOOP_INPUTS[kern]:
                args = (seed.args[0],) + tuple(IntValue(v) for v in vals)
                cases.append((kern, m, TestCase(args, seed.rng_seed)))
        mm = rc.load_harness(REPO / "paper_2603_05725_b200" / "workloads" / "matmul.man")
        for mv, nv in MATMUL_LOOPS:
            s = mm.seed(1)
            args = list(s.args)
            args[3], args[4] = IntValue(mv), IntValue(nv)
            cases.append(("matmul", mm, TestCase(tuple(args), s.rng_seed)))
        for budget in LOOP_BUDGETS:
            for kern, m, tc in cases:
                image = DeviceMemoryImage()
                runner = rc.PhaseRunner(m, image, instruction_budget=budget, diff_readback=True)
                runner.run_phase(rc.INIT, m.seed(1), iteration=0)
                runner.mark_baseline()
                cov = CoverageMap.for_program(m.program)
                res = runner.run_phase(rc.COMPUTE, tc, coverage=cov, iteration=1)
                out["inputs"].setdefault(kern, []).append({
                    "budget": budget, "testcase": serialize_testcase(tc, with_id=False), "status": res.status,
                    "retired": res.retired, "report": res.report.to_line() if res.report else None,
                    "readouts": {k: v.hex() for k, v in res.readouts.items()}, "edges": edges_json(cov)})
        for kern in ("spin", "spin2"):
            m = rc.load_harness(Path(tmp) / f"{kern}.man")
            out["campaigns"][kern] = batched(m, **LOOP_CAMPAIGN)
    return out


# Loop nests with loads and stores (the JIT's nest summaries, csrc/jit.cu
# analyse_nest) on the C2 matmul kernel: row loops whose cols / inner loops touch
# the same addresses every row (a zero or wrapping leading dimension: i*lda*4 and
# i*ldc*4 are 0 mod 2^32 for every row step of 8), to the budget at every position
# of a row trip (budgets 10^6 + k) or to the row exit; and nests whose guards fail
# (a stride that moves the accesses every row), ending at the budget or in an
# out-of-bounds store.  (m, n, k, lda, ldb, ldc)
M31N = 1 << 31
NEST_INPUTS = [
    ((1 << 31) - 1, 8, 0, 8, 8, -M31N),        # stores only, wrapping ldc: summarized to the budget
    (16515080, 8, 8, 0, 8, 0),                 # loads + stores, zero lda / ldc
    (15925256, 8, 8, -M31N, 8, -M31N),         # loads + stores, wrapping lda / ldc
    (40000, 8, 0, 8, 8, 0),                    # exits at the row test before the budget
    (4000, 8, 8, 0, 8, 0),                     # exits, loads + stores
    (8000, 8, -5, 8, 8, -M31N),                # exits, inner loop never entered
    ((1 << 31) - 1, 8, 8, 8, 8, 0),            # guard fails (lda moves the A row): plain execution
    ((1 << 31) - 1, 8, 0, 8, 8, 1),            # guard fails (ldc = 1): out-of-bounds store
]
NEST_BUDGETS = [10 ** 6 + k for k in range(0, 700, 97)] + [200003]


def nests():
    mm = rc.load_harness(REPO / "paper_2603_05725_b200" / "workloads" / "matmul.man")
    out = {"inputs": NEST_INPUTS, "budgets": NEST_BUDGETS, "records": []}
    for budget in NEST_BUDGETS:
        for vals in NEST_INPUTS:
            s = mm.seed(1)
            args = list(s.args)
            for j, v in enumerate(vals):
                args[3 + j] = IntValue(v)
            tc = TestCase(tuple(args), s.rng_seed)
            image = DeviceMemoryImage()
            runner = rc.PhaseRunner(mm, image, instruction_budget=budget, diff_readback=True)
            runner.run_phase(rc.INIT, mm.seed(1), iteration=0)
            runner.mark_baseline()
            cov = CoverageMap.for_program(mm.program)
            res = runner.run_phase(rc.COMPUTE, tc, coverage=cov, iteration=1)
            out["records"].append({
                "budget": budget, "testcase": serialize_testcase(tc, with_id=False), "status": res.status,
                "retired": res.retired, "report": res.report.to_line() if res.report else None,
                "readouts": {k: v.hex() for k, v in res.readouts.items()}, "edges": edges_json(cov)})
    return out


# Phase features beyond the bundled harnesses (campaign.py:483-561, 723-762):
# kernels storing >= 4 KB per exec into an INIT (`buf:`) buffer, an INIT-phase
# launch (with an array argument materialized in INIT), a TERM-phase launch that
# reports (iteration -1) plus an idempotent double free, and a COMPUTE
# `copy_in <buf> arg:N` of an array argument after a launch modified it.
FEATURES_SIR = """\
kernel fill(ws:ptr.global, x:ptr.global, n:i32, k:i32) regs=12
  sreg %r2, tid
  sreg %r3, ntid
  sreg %r4, ctaid
  mul %r5, %r4, %r3
  add %r5, %r5, %r2
  mul %r6, %r5, %r0
  mul %r6, %r6, 4
  mov %a2, %a0
  add %a2, %a2, %r6
  mov %r7, 0
loop:
  setp.ge %p0, %r7, %r0
  bra %p0, done
  ld.global.b32 %r8, [%a2]
  add %r8, %r8, %r1
  st.global.b32 [%a2], %r8
  add %a2, %a2, 4
  add %r7, %r7, 1
  bra loop
done:
  ld.global.f32 %f0, [%a1]
  exit

kernel prep(tab:ptr.global, x:ptr.global) regs=8
  sreg %r0, tid
  sreg %r1, ntid
  ld.global.b32 %r4, [%a1]
top:
  setp.ge %p0, %r0, 1024
  bra %p0, fin
  mul %r2, %r0, 4
  mov %a2, %a0
  add %a2, %a2, %r2
  ld.global.b32 %r3, [%a2]
  mul %r3, %r3, 3
  add %r3, %r3, %r4
  st.global.b32 [%a2], %r3
  add %r0, %r0, %r1
  bra top
fin:
  st.global.b32 [%a1], %r1
  exit

kernel use(tab:ptr.global, x:ptr.global, n:i32) regs=8
  mul %r1, %r0, 4
  mov %a2, %a0
  add %a2, %a2, %r1
  ld.global.b32 %r2, [%a2]
  setp.lt %p0, %r2, 100
  bra %p0, small
  st.global.b32 [%a1], %r2
  exit
small:
  st.global.b32 [%a1+4], %r2
  exit

kernel check(tab:ptr.global, n:i32) regs=4
  mul %r1, %r0, 4
  mov %a1, %a0
  add %a1, %a1, %r1
  ld.global.b32 %r2, [%a1]
  exit

kernel scribble(x:ptr.global, n:i32) regs=6
  mov %r1, 0
  mov %a1, %a0
s_top:
  setp.ge %p0, %r1, %r0
  bra %p0, s_end
  st.global.b32 [%a1], 7
  add %a1, %a1, 4
  add %r1, %r1, 1
  bra s_top
s_end:
  exit

kernel cmp(c:ptr.global, x:ptr.global, n:i32) regs=10
  mov %r1, 0
  mov %r2, 0
  mov %a2, %a0
  mov %a3, %a1
c_top:
  setp.ge %p0, %r1, 4
  bra %p0, c_end
  ld.global.b32 %r3, [%a2]
  ld.global.b32 %r4, [%a3]
  setp.eq %p1, %r3, %r4
  bra !%p1, c_next
  add %r2, %r2, 1
c_next:
  add %a2, %a2, 4
  add %a3, %a3, 4
  add %r1, %r1, 1
  bra c_top
c_end:
  setp.gt %p2, %r2, 2
  bra %p2, c_same
  exit
c_same:
  st.global.b32 [%a0], %r2
  exit
"""

FEATURE_MANIFESTS = {
    "bufwrite": ("argspec x ptr global f32 count=16 seed=seq flo=-4 fhi=4\n"
                 "argspec n i32 seed=160 lo=0 hi=400\n"
                 "argspec k i32 seed=3 lo=-5 hi=5\n\n"
                 "init:\n  alloc ws global 65536\n  copy_in ws seq32:16384\n"
                 "compute:\n  launch fill grid=2 block=4 args=buf:ws,arg:0,arg:1,arg:2\n  copy_out ws 64\n"
                 "term:\n  free ws\n"),
    "initlaunch": ("argspec x ptr global i32 count=4 seed=seq lo=0 hi=9\n"
                   "argspec n i32 seed=5 lo=0 hi=1100\n\n"
                   "init:\n  alloc tab global 4096\n  copy_in tab seq32:1024\n"
                   "  launch prep grid=1 block=4 args=buf:tab,arg:0\n  copy_out arg:0\n"
                   "compute:\n  launch use grid=1 block=1 args=buf:tab,arg:0,arg:1\n  copy_out arg:0\n"
                   "term:\n  free tab\n"),
    "termlaunch": ("argspec x ptr global i32 count=4 seed=seq lo=0 hi=9\n"
                   "argspec n i32 seed=5 lo=0 hi=1100\n\n"
                   "init:\n  alloc tab global 4096\n  copy_in tab seq32:1024\n"
                   "compute:\n  launch use grid=1 block=1 args=buf:tab,arg:0,arg:1\n"
                   "term:\n  launch check grid=1 block=1 args=buf:tab,lit:i32:1024\n  free tab\n  free tab\n"),
    "copyarg": ("argspec x ptr global i32 count=4 seed=seq lo=0 hi=9\n"
                "argspec n i32 seed=2 lo=0 hi=4\n\n"
                "compute:\n  alloc cbuf global 256\n  launch scribble grid=1 block=1 args=arg:0,arg:1\n"
                "  copy_in cbuf arg:0\n  launch cmp grid=1 block=1 args=buf:cbuf,arg:0,arg:1\n  free cbuf\n"
                "  copy_out arg:0\n"),
}
FEATURE_CAMPAIGN = dict(master_seed=11, iterations=600, round_size=128)


def features():
    import tempfile
    out = {"kernel": FEATURES_SIR, "manifests": {}, "campaigns": {}, "fuzzloops": {},
           "campaign_config": FEATURE_CAMPAIGN}
    with tempfile.TemporaryDirectory() as tmp:
        (Path(tmp) / "features.sir").write_text(FEATURES_SIR)
        for name, body in FEATURE_MANIFESTS.items():
            man = "program features.sir\n\n" + body
            out["manifests"][name] = man
            (Path(tmp) / f"{name}.man").write_text(man)
            m = rc.load_harness(Path(tmp) / f"{name}.man")
            out["campaigns"][name] = batched(m, **FEATURE_CAMPAIGN)
            d = Path(tmp) / f"out-{name}"
            s = rc.fuzz_loop(m, rc.CampaignConfig(master_seed=5, iterations=300, out_dir=d))
            out["fuzzloops"][name] = {
                "summary": s.to_rec(), "findings": (d / "findings.txt").read_text(),
                "coverage_rec": (d / "coverage.rec").read_text(),
                "corpus": sorted(p.name for p in (d / "corpus").iterdir()),
                "crashes": sorted(p.name for p in (d / "crashes").iterdir())}
    return out


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def main():
    import tempfile
    which = sys.argv[1:] or ["assets", "variants", "sampled", "batched", "fuzzloop", "workloads", "traces",
                             "errors", "loops", "features", "nests"]
    if "assets" in which:
        (HERE / "bench_assets.json").write_text(_dump(assets()))
    if "variants" in which:
        (HERE / "ref_variants.json").write_text(_dump(variants()))
    if "sampled" in which:
        (HERE / "ref_sampled.json").write_text(_dump(sampled()))
    if "batched" in which:
        data = {"config": BATCH_CFG, "keybase": KEYBASE, "runs": batched_all()}
        (HERE / "ref_batched.json").write_text(_dump(data))
    if "fuzzloop" in which:
        with tempfile.TemporaryDirectory() as tmp:
            (HERE / "ref_fuzzloop.json").write_text(_dump(fuzzloops(tmp)))
    if "workloads" in which:
        (HERE / "ref_workloads.json").write_text(_dump(workloads()))
    if "traces" in which:
        (HERE / "ref_traces.json").write_text(_dump(traces()))
    if "features" in which:
        (HERE / "ref_features.json").write_text(_dump(features()))
    if "loops" in which:
        (HERE / "ref_loops.json").write_text(_dump(loops()))
    if "nests" in which:
        (HERE / "ref_nests.json").write_text(_dump(nests()))
    if "errors" in which:
        with tempfile.TemporaryDirectory() as tmp:
            (HERE / "ref_errors.json").write_text(_dump(errors(tmp)))


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
