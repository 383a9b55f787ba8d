"""ORACLE (test infrastructure): phase runner, scheduler and campaign loops.

Restates ``simt_forge/campaign.py``: ``PhaseRunner`` :412-561 (lazy array
materialization :440-479, host-op loop :483-561), ``Corpus``/``schedule_next``
:567-603, ``fuzz_loop`` amortized path :683-762 and ``_absorb_iteration``
:825-846, ``execute_once`` :872-891.

Two loop drivers:

* ``sequential_loop`` — the reference ``fuzz_loop`` (one worker stream
  ``Stream(seed, 1000 + w)``, live corpus).  Used to pin this oracle against
  the reference's own campaign outputs (tests/golden).
* ``batched_loop`` — the batched-round contract the GPU implements
  (SURVEY.md §8(c) "Level A"): input ``it`` draws from its own stream
  ``Stream(seed, KEYBASE + it)``; parents are scheduled from the corpus as it
  stood at the start of the input's round; everything else (rotation counts,
  alloc ids, absorption, admission, stop) happens in ``it`` order exactly as in
  the reference loop.  Emits one record per executed input for parity tests.
"""

from __future__ import annotations

import struct

import numpy as np

from paper_2603_05725_b200.coverage import CoverageMap, new_edges_since
from paper_2603_05725_b200.findings import BugClass, FindingsLog
from paper_2603_05725_b200.manifest import COMPUTE, INIT, TERM
from paper_2603_05725_b200.sir import ScalarType
from paper_2603_05725_b200.testcase import ArrayValue, FloatValue, IntValue

from .execute import launch
from .memory import Image, InvalidFreeError, MemCfg, OutOfSpaceError, invalid_free_report
from .mutate import draw_picks, finish_child
from .rng import OracleStream

KEYBASE = 1 << 32   # per-input stream ids: KEYBASE + it (clear of 1000+w / 2000+w)


class PhaseResult:
    __slots__ = ("status", "report", "retired", "launches", "readouts")

    def __init__(self):
        self.status, self.report, self.retired, self.launches, self.readouts = "ok", None, 0, 0, {}


def scalar_bytes(v) -> bytes:
    if isinstance(v, IntValue):
        return struct.pack("<i", v.value)
    if isinstance(v, FloatValue):
        return struct.pack("<I", v.bits)
    return v.data


class Runner:
    def __init__(self, manifest, img: Image, budget=1_000_000, diff_readback=False):
        self.m, self.img, self.budget, self.diff = manifest, img, budget, diff_readback
        self.named = {}
        self.base_named = None
        self.mat = {}

    def mark_baseline(self):
        self.base_named = dict(self.named)

    def reset(self):
        self.named = dict(self.base_named)
        self.mat = {}

    def _materialize(self, k, v: ArrayValue):
        size = v.size_override if v.size_override is not None else len(v.data)
        if size <= 0:
            addr, aid = self.img.alloc(v.space, 0, f"arg{k}")
            payload = b""
        else:
            addr, aid = self.img.alloc(v.space, size, f"arg{k}")
            payload = v.data[:size]
        rep = self.img.copy_in(addr, payload) if payload else None
        self.mat[k] = (addr, aid, len(v.data))
        return addr, aid, rep

    def run(self, phase, tc, coverage=None, iteration=-1) -> PhaseResult:
        out = PhaseResult()
        img = self.img
        if phase == COMPUTE:
            self.mat = {}
        for op in self.m.phases[phase]:
            kd = op.kind
            if kd == "alloc":
                if op.size <= 0:
                    raise ValueError(f"allocation size must be positive, got {op.size}")
                self.named[op.name] = img.alloc(op.space, op.size, op.name)
            elif kd == "copy_in":
                addr, _ = self.named[op.name]
                form, pl = op.source
                if form == "zeros":
                    data = bytes(int(pl, 0))
                elif form == "seq32":
                    data = np.arange(int(pl, 0), dtype="<u4").tobytes()
                elif form == "hex":
                    data = bytes.fromhex(pl)
                else:
                    data = scalar_bytes(tc.args[int(pl)])
                rep = img.copy_in(addr, data)
                if rep is not None:
                    rep.iteration = iteration
                    out.status, out.report = "finding", rep
                    return out
            elif kd == "copy_out":
                if op.arg_ref >= 0:
                    if phase == COMPUTE and not self.diff:
                        continue
                    if op.arg_ref not in self.mat:
                        continue
                    addr, _, n = self.mat[op.arg_ref]
                    data, rep = img.copy_out(addr, n)
                    key = f"arg{op.arg_ref}"
                else:
                    addr, _ = self.named[op.name]
                    data, rep = img.copy_out(addr, op.size)
                    key = op.name
                if rep is not None:
                    rep.iteration = iteration
                    out.status, out.report = "finding", rep
                    return out
                out.readouts[key] = data
            elif kd == "free":
                addr, _ = self.named[op.name]
                try:
                    img.free(addr)
                except InvalidFreeError as exc:
                    if phase == TERM and exc.reason == "allocation already freed":
                        continue
                    out.status, out.report = "finding", invalid_free_report(img, addr, iteration)
                    return out
            elif kd == "launch":
                kern = self.m.program.kernels[op.kernel]
                args = []
                for b, p in zip(op.bindings, kern.params):
                    if b[0] == "lit_i32":
                        args.append((ScalarType.I32, b[1], None))
                    elif b[0] == "lit_f32":
                        args.append((ScalarType.F32, b[1], None))
                    elif b[0] == "buf":
                        addr, aid = self.named[b[1]]
                        args.append((ScalarType.PTR, addr, aid))
                    else:
                        v = tc.args[b[1]]
                        if isinstance(v, ArrayValue):
                            if b[1] in self.mat:
                                addr, aid, _ = self.mat[b[1]]
                            else:
                                addr, aid, rep = self._materialize(b[1], v)
                                if rep is not None:
                                    rep.iteration = iteration
                                    out.status, out.report = "finding", rep
                                    return out
                            args.append((ScalarType.PTR, addr + v.base_offset, aid))
                        elif isinstance(v, IntValue):
                            args.append((ScalarType.I32, v.value, None))
                        else:
                            args.append((ScalarType.F32, v.value, None))
                res = launch(self.m.program, img, op.kernel, op.grid, op.block, args,
                             coverage=coverage, budget=self.budget, iteration=iteration)
                out.retired += res.retired
                out.launches += 1
                if res.status == "SANITIZER_STOP":
                    out.status, out.report = "finding", res.report
                    return out
                if res.status == "BUDGET_EXHAUSTED":
                    out.status = "budget"
                    return out
        return out


class Entry:
    __slots__ = ("tc", "admitted_iteration", "is_seed")

    def __init__(self, tc, it, is_seed):
        self.tc, self.admitted_iteration, self.is_seed = tc, it, is_seed


def schedule_next(entries, rng, it, window=256, weight=4.0):
    ws = [weight if (not e.is_seed and it - e.admitted_iteration <= window) else 1.0 for e in entries]
    return rng.weighted_choice(entries, ws).tc


class OracleCampaign:
    """Result container (reference-shaped fields)."""

    def __init__(self):
        self.findings = FindingsLog()
        self.coverage = None
        self.corpus: list = []
        self.records: list = []
        self.stop_reason = "iterations"
        self.executed = 0


def _edges_of(delta: CoverageMap):
    return {k: sorted([s, d, c] for (s, d), c in v.items()) for k, v in delta.edge_counts.items() if v}


def run_loop(manifest, *, master_seed=1, iterations=1000, batched=True, round_size=256,
             stop_on_first_finding=False, stop_bug_class=None, budget=1_000_000,
             mem_cfg: MemCfg | None = None, max_ops=3, granule=4, redzone=32,
             window=256, weight=4.0, keep_records=True, extra_seeds=(), fanout=0, on_exec=None):
    """Shared body of ``sequential_loop`` / ``batched_loop``.  ``on_exec()``
    (bench CPU baseline only) is called after every input; True stops the loop."""
    specs = manifest.argspecs
    res = OracleCampaign()
    gcov = CoverageMap.for_program(manifest.program)
    res.coverage = gcov
    seed_tc = manifest.seed(master_seed)
    corpus = [Entry(seed_tc, 0, True)] + [Entry(t, 0, True) for t in extra_seeds]
    res.corpus = corpus
    img = Image(mem_cfg or MemCfg())
    runner = Runner(manifest, img, budget)
    init = runner.run(INIT, seed_tc, iteration=0)
    if init.status != "ok":
        raise RuntimeError(f"init phase failed on the seed input: {init.status}")
    runner.mark_baseline()
    snap = img.snapshot()
    counts: dict = {}
    worker = OracleStream(master_seed, 1000)
    want = None
    if stop_bug_class is not None:
        want = stop_bug_class.value if isinstance(stop_bug_class, BugClass) else str(stop_bug_class)
    round_entries = list(corpus)
    for it in range(1, iterations + 1):
        if batched and (it - 1) % round_size == 0:
            round_entries = list(corpus)
        img.restore(snap)
        runner.reset()
        rec = {"it": it}
        if it == 1:
            child = seed_tc
            rec["parent"] = -1
        else:
            s = OracleStream(master_seed, KEYBASE + it) if batched else worker
            pool = round_entries if batched else corpus
            if fanout:   # fixed fan-out (BASELINE.json configs[3]): no scheduling draw
                pidx = ((it - 1) // fanout) % len(pool)
                parent = pool[pidx].tc
            else:
                parent = schedule_next(pool, s, it, window, weight)
                pidx = next(i for i, e in enumerate(pool) if e.tc is parent)
            rec["parent"] = pidx
            picks = draw_picks(specs, s, max_ops)
            child = finish_child(parent, picks, counts, s, granule, redzone)
        delta = gcov.fresh()
        first_id = img.next_id
        try:
            out = runner.run(COMPUTE, child, coverage=delta, iteration=it)
        except OutOfSpaceError as exc:
            rec["fatal"] = str(exc)
            res.records.append(rec)
            raise
        res.executed += 1
        fresh = new_edges_since(delta, gcov)
        gcov.merge_from(delta)
        rec.update(child=child, status=out.status, retired=out.retired, allocs=img.next_id - first_id,
                   edges=_edges_of(delta), entered=sorted(k for k, v in delta.entered.items() if v),
                   report=out.report.to_line() if out.report else None, admitted=False)
        stop = None
        if out.report is not None:
            out.report.iteration = it
            rec["report"] = out.report.to_line()
            res.findings.add(out.report)
            if stop_on_first_finding:
                stop = "first_finding"
            elif want is not None and out.report.bug_class.value == want:
                stop = f"bug_class:{want}"
        elif fresh and it != 1:
            corpus.append(Entry(child, it, False))
            rec["admitted"] = True
        if keep_records:
            res.records.append(rec)
        if stop:
            res.stop_reason = stop
            break
        if on_exec is not None and on_exec():
            res.stop_reason = "on_exec"
            break
    return res


def sequential_loop(manifest, **kw):
    return run_loop(manifest, batched=False, **kw)


def batched_loop(manifest, **kw):
    return run_loop(manifest, batched=True, **kw)


def execute_once(manifest, tc, *, budget=1_000_000, diff_readback=False, coverage=None,
                 image_seed=1, mem_cfg=None):
    img = Image(mem_cfg or MemCfg())
    runner = Runner(manifest, img, budget, diff_readback)
    seed_tc = manifest.seed(image_seed)
    if runner.run(INIT, seed_tc, iteration=0).status != "ok":
        raise RuntimeError("init phase failed")
    runner.mark_baseline()
    return runner.run(COMPUTE, tc, coverage=coverage, iteration=0), img
