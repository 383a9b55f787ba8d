"""``fuzz_loop`` with the reference's signature and result types, on the GPU.

Drop-in for ``simt_forge.campaign.fuzz_loop`` (campaign.py:683-822): same
``CampaignConfig`` fields (plus ``round_size`` and ``device``), same
``CampaignSummary`` (findings as a ``FindingsLog`` of ``BugReport``,
``CoverageMap``, ``Corpus`` of ``TestCase``), same output directory layout.

Semantics are the batched-round contract: iterations are
processed in rounds of ``round_size`` inputs; input ``it`` draws from its own
Philox stream ``(master_seed, 2**32 + it)`` and schedules its parent from the
corpus as it stood at its round's start.  Everything else (rotation counts,
alloc ids, absorption order, admission, dedupe, stop rules) follows the
reference in ``it`` order, so results equal the reference functions driven
the same way (tests/golden/make_golden.py ``batched``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from pathlib import Path

from .baseline import InitFailure, MemConfig
from .coverage import build_report, render_text, report_to_rec
from .engine import DeviceCampaign, MutationConfig
from .findings import BugClass, FindingsLog
from .hooks import ExecHooks, TraceHooks, dispatch  # noqa: F401  (re-export)
from .lowering import LoweringError
from .manifest import HarnessManifest, load_harness  # noqa: F401  (re-export)
from .interop import as_config, as_manifest, as_testcase
from .testcase import argspec_digest, serialize_testcase


class CampaignFatalError(Exception):
    pass


@dataclass
class CorpusEntry:
    tc: object
    admitted_iteration: int
    is_seed: bool


@dataclass
class Corpus:
    entries: list = field(default_factory=list)

    @property
    def seeds(self) -> int:
        return sum(1 for e in self.entries if e.is_seed)

    @property
    def interesting(self) -> int:
        return sum(1 for e in self.entries if not e.is_seed)


@dataclass
class CampaignConfig:
    master_seed: int = 1
    iterations: int = 1000
    workers: int = 1
    mode: str = "amortized"
    out_dir: Path | None = None
    stop_on_first_finding: bool = False
    stop_bug_class: BugClass | str | None = None
    max_wall_seconds: float | None = None
    instruction_budget: int = 1_000_000
    mem_config: MemConfig = field(default_factory=MemConfig)
    mutation: MutationConfig = field(default_factory=MutationConfig)
    admission_window: int = 256
    recent_weight: float = 4.0
    diff_readback: bool = False
    hooks: object = None
    round_size: int = 65536
    pipeline_depth: int = 24
    device: str | None = None
    # shard every round over the ranks of the initialized torch.distributed group
    # (one process per GPU, per-round merge, shard.py); results do not depend on it
    distributed: bool = False
    # "batched": the batched-round contract (per-input streams, parents
    # from the round-start corpus) -- the throughput path; "sequential": the
    # reference fuzz_loop's own discipline (one worker stream, live corpus), rounds
    # generated in order on the device and cut after each admission -- results
    # identical to the reference fuzz_loop, output directories byte for byte
    discipline: str = "batched"
    # extensions for BASELINE.json configs 3-4 (not reference fields): the 16 MiB
    # context-sensitive hashed coverage map (2^ctx_map_bits one-byte slots, a derived
    # view; summary.context_map_slots), extra seed test cases added to the corpus
    # after the manifest seed, and fixed fan-out (input it mutates round-corpus entry
    # ((it - 1) // fanout) mod n instead of schedule_next); soft_cap: retired
    # instructions before an input moves to the long-input pass (None = default)
    ctx_map_bits: int = 0
    extra_seeds: tuple = ()
    fanout: int = 0
    soft_cap: int | None = None
    # opt-in: children of a round with the same parent and the same set of ops run
    # once and share the verdict (results identical; fewer executions than inputs --
    # off by default, and off in the bench's headline figures)
    dedupe_inputs: bool = False


@dataclass
class CampaignSummary:
    master_seed: int
    iterations_requested: int
    iterations_executed: int
    workers: int
    mode: str
    program_digest: str
    manifest_digest: str
    argspec_digest: str
    findings: FindingsLog
    coverage: object
    corpus: Corpus
    stop_reason: str
    init_runs: int
    compute_runs: int
    term_runs: int
    wall_seconds: float
    out_dir: Path | None

    @property
    def execs_per_second(self) -> float:
        return self.compute_runs / self.wall_seconds if self.wall_seconds > 0 else 0.0

    def to_reference(self, sf, reference_manifest):
        """(FindingsLog, CoverageMap, Corpus) as the reference package's own types
        (``sf`` = the imported ``simt_forge`` module; interop.summary_to_reference)."""
        from .interop import summary_to_reference
        return summary_to_reference(self, sf, reference_manifest.program)

    def to_rec(self) -> str:
        return "\n".join([
            "summary v1",
            f"master_seed={self.master_seed} workers={self.workers} mode={self.mode}",
            f"iterations_requested={self.iterations_requested} iterations_executed={self.iterations_executed}",
            f"program={self.program_digest} manifest={self.manifest_digest} argspec={self.argspec_digest}",
            f"findings_unique={len(self.findings)} findings_total={self.findings.total}",
            f"corpus_seeds={self.corpus.seeds} corpus_interesting={self.corpus.interesting}",
            f"init_runs={self.init_runs} compute_runs={self.compute_runs} term_runs={self.term_runs}",
            f"stop={self.stop_reason}",
        ]) + "\n"


def _worker_ranges(total: int, workers: int):
    base, rem = divmod(total, workers)
    out, start = [], 1
    for w in range(workers):
        n = base + (1 if w < rem else 0)
        out.append(range(start, start + n))
        start += n
    return out


def _device_campaign(manifest, config: CampaignConfig, comm) -> DeviceCampaign:
    return DeviceCampaign(manifest, master_seed=config.master_seed, mem=config.mem_config, comm=comm,
                          mutation=config.mutation, budget=config.instruction_budget,
                          window=config.admission_window, recent_weight=config.recent_weight,
                          diff_readback=config.diff_readback, stop_on_first_finding=config.stop_on_first_finding,
                          stop_bug_class=config.stop_bug_class, device=config.device,
                          ids_reset_per_input=config.mode == "reinit",
                          sequential=config.discipline == "sequential", ctx_map_bits=config.ctx_map_bits,
                          extra_seeds=tuple(as_testcase(t) for t in config.extra_seeds), fanout=config.fanout,
                          soft_cap=config.soft_cap, dedupe=config.dedupe_inputs)


def fuzz_loop(manifest, config: CampaignConfig) -> CampaignSummary:
    # the reference's own objects are accepted as they are (interop.py)
    manifest, config = as_manifest(manifest), as_config(config)
    if config.mode not in ("amortized", "reinit"):
        raise CampaignFatalError(f"unknown mode {config.mode!r}")
    if config.workers < 1 or config.iterations < 1:
        raise CampaignFatalError("workers and iterations must be >= 1")
    if config.discipline not in ("batched", "sequential"):
        raise CampaignFatalError(f"unknown discipline {config.discipline!r}")
    hooks = config.hooks
    if config.mode == "reinit" and any(op.kind not in ("free", "sync") for op in manifest.phases["term"]):
        # reinit runs TERM after every input on that input's post-COMPUTE state
        raise LoweringError("reinit mode: TERM phases other than frees are not lowered")
    out_dir = Path(config.out_dir) if config.out_dir is not None else None
    specs = manifest.argspecs
    if out_dir is not None:
        (out_dir / "corpus").mkdir(parents=True, exist_ok=True)
        (out_dir / "crashes").mkdir(parents=True, exist_ok=True)
        (out_dir / "program.sir").write_text(manifest.program_text)
        (out_dir / "harness.man").write_text(manifest.portable_text("program.sir"))
    t0 = time.perf_counter()
    deadline = t0 + config.max_wall_seconds if config.max_wall_seconds else None
    comm = None
    if config.distributed and hooks is not None:
        raise LoweringError("hooks are per-process; trace a campaign on one device")
    if config.distributed:
        from .shard import RoundComm
        comm = RoundComm()
    # the seed corpus entry is written before anything can fail (campaign.py:700-703)
    if out_dir is not None:
        _write_corpus_entry(out_dir, manifest.seed(config.master_seed), specs)
    stop_reason = "iterations"
    executed = 0
    init_runs = term_runs = 0
    dc = None
    try:
        t_setup = time.perf_counter()
        try:
            dc = _device_campaign(manifest, config, comm)
        except InitFailure as e:   # campaign.py:723-725: the init phase failed on the seed input
            raise CampaignFatalError(str(e)) from e
        t_setup = time.perf_counter() - t_setup
        for w, rng_ in enumerate(_worker_ranges(config.iterations, config.workers)):
            if stop_reason != "iterations":
                break
            dc.new_worker(w)  # fresh rotation counts + alloc ids (one image per worker)
            if config.mode == "amortized":
                init_runs += 1
            state = {"stop": None}

            def on_round(res):
                nonlocal executed, init_runs, term_runs
                executed += res.executed
                if config.mode == "reinit":
                    init_runs += res.executed
                    term_runs += res.executed
                if out_dir is not None:
                    for tc, _, _ in dc.host_entries[on_round.mirrored:]:
                        _write_corpus_entry(out_dir, tc, specs)
                    on_round.mirrored = len(dc.host_entries)
                    if res.new_keys:
                        tcs = dc.child_testcases([i for i, _ in res.new_keys], res.slot)
                        for (i, rep), tc in zip(res.new_keys, tcs):
                            _write_crash(out_dir, rep, tc, specs, manifest)
                if hooks is not None and res.executed:
                    # the round's inputs once more through the device trace mode, events
                    # replayed to the hooks in iteration order (hooks.py)
                    k = min(res.executed, res.slot.n)
                    tcs = dc.child_testcases(list(range(k)), res.slot)
                    for out in dc.execute_testcases(tcs, iteration0=res.slot.it0, trace=True):
                        dispatch(hooks, out["events"])
                if res.stop is not None:
                    want = config.stop_bug_class
                    state["stop"] = ("first_finding" if config.stop_on_first_finding else
                                     f"bug_class:{getattr(want, 'value', want)}")

            on_round.mirrored = len(dc.host_entries)
            clock = {"expired": False}

            def should_continue():
                # wall-clock limit checked before every round submission (campaign.py:733-735);
                # rounds already in flight are finalized.  Sharded: the ranks agree (MAX).
                if deadline is not None and not clock["expired"]:
                    late = time.perf_counter() > deadline
                    if dc.comm.world > 1:
                        late = bool(dc.comm.all_gather_object(late).count(True))
                    clock["expired"] = late
                return not clock["expired"]

            dc.run_rounds(rng_.start, rng_.stop, config.round_size,
                          depth=1 if hooks is not None else config.pipeline_depth,
                          on_round=on_round, should_continue=should_continue)
            if clock["expired"] and state["stop"] is None:
                stop_reason = "wall_clock"
            if state["stop"] is not None:
                stop_reason = state["stop"]
            if config.mode == "amortized":
                # TERM once per worker on the restored state (campaign.py:756-762)
                rep = dc.run_term()
                term_runs += 1
                if rep is not None and dc.findings.add(rep) and out_dir is not None:
                    _write_crash(out_dir, rep, dc.seed_tc, specs, manifest)
    except CampaignFatalError:
        if out_dir is not None:
            (out_dir / "FAILED").write_text("campaign fatal\n")
        if dc is not None:
            dc.close()
        raise
    except BaseException:
        if dc is not None:    # release the round buffers now, not at garbage collection
            dc.close()
        raise
    if dc.round_log is not None:
        dc.round_log.append(("loop_end", -1, time.perf_counter()))
    wall = time.perf_counter() - t0
    corpus = Corpus([CorpusEntry(tc, adm, seed) for tc, adm, seed in dc.host_entries])
    cov = dc.coverage_map()
    summary = CampaignSummary(config.master_seed, config.iterations, executed, config.workers, config.mode,
                              manifest.program_digest, manifest.digest, argspec_digest(specs), dc.findings,
                              cov, corpus, stop_reason, init_runs, executed, term_runs, wall, out_dir)
    if out_dir is not None:
        rep = build_report(cov)
        (out_dir / "coverage.txt").write_text(render_text(rep))
        (out_dir / "coverage.rec").write_text(report_to_rec(rep))
        (out_dir / "findings.txt").write_text(dc.findings.render_text())
        (out_dir / "summary.rec").write_text(summary.to_rec())
        (out_dir / "timing.rec").write_text(
            f"timing v1\nwall_seconds={wall:.6f} execs_per_second={summary.execs_per_second:.2f}\n")
    # host<->device traffic of the campaign (not a reference field; bench e2e accounting)
    summary.device_transfer = {"h2d_bytes": dc.h2d_bytes, "d2h_bytes": dc.d2h_bytes, "rounds": dc.rounds,
                               "setup_s": t_setup}
    if config.ctx_map_bits:
        summary.context_map_slots = dc.ctx_map_slots()
    if dc.round_log is not None:
        dc.round_log.append(("summary", -1, time.perf_counter()))
        summary.device_transfer["round_log"] = dc.round_log
    dc.close()
    if dc.round_log is not None:
        dc.round_log.append(("closed", -1, time.perf_counter()))
    return summary


def _write_corpus_entry(out_dir: Path, tc, specs) -> None:
    (out_dir / "corpus" / f"{tc.id}.tc").write_text(serialize_testcase(tc, specs))


def _write_crash(out_dir: Path, report, tc, specs, manifest) -> None:
    extra = [f"crash class={report.bug_class.value} dedupe={report.dedupe_key} kernel={report.kernel} "
             f"iid={report.iid} addr=0x{report.address:x} width={report.width} iteration={report.iteration}",
             f"origin harness=../harness.man program={manifest.program_digest} manifest={manifest.digest}"]
    (out_dir / "crashes" / f"{report.dedupe_key}.tc").write_text(serialize_testcase(tc, specs, extra=extra))
