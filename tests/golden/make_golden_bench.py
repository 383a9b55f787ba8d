"""Golden fixtures at the BENCH configuration, made by running the REAL reference here.

The batched-round contract on the reference's own functions
(`schedule_next`, `mutate_testcase` with one shared `MutationSchedule`,
`PhaseRunner.run_phase(COMPUTE)` on the restored post-INIT image,
`new_edges_since` / `merge_from` / `FindingsLog.add` / `Corpus.admit` in input
order), exactly as `make_golden.batched`, but at the round sizes the bench and
the C5 mix use.  Inputs of a round are independent given the round-start
corpus and rotation counts, so their COMPUTE phases run in a process pool;
mutation and absorption stay sequential, in input order.

Allocation ids are campaign-scoped (`device_memory.py:279`): each worker runs an
input with its image's id counter at a placeholder and the ids in its report are
shifted to the sequential value (round-start id + allocations of earlier
inputs) during absorption.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_bench.py [c2] [c5]

Writes (gzip JSON, committed):
  ref_bench_c2.json.gz  workloads/matmul.man, master_seed 11, R = 2^20 (bench.py's default):
                        round 1 in full (per-1024-input block hashes of the
                        records, the first 20,000 records verbatim, findings /
                        coverage / corpus after the round) and the first 4,096
                        records of round 2
  ref_bench_c5.json.gz  dot, amax, rotm, master_seed 11, R = 2^14, two full
                        rounds each (block hashes, first 2,000 records,
                        per-round findings / coverage / corpus)
"""

from __future__ import annotations

import dataclasses
import gzip
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

from make_golden import KEYBASE, digest, edges_json  # noqa: E402
from simt_forge import bench as rb  # noqa: E402
from simt_forge import campaign as rc  # noqa: E402
from simt_forge.coverage import CoverageMap, build_report, new_edges_since, report_to_rec  # noqa: E402
from simt_forge.device_memory import DeviceMemoryImage  # noqa: E402
from simt_forge.mutation import MutationSchedule, mutate_testcase  # noqa: E402
from simt_forge.rng import Stream  # noqa: E402

PLACEHOLDER = 1 << 40      # worker-side alloc id base; shifted during absorption
BLOCK = 1024


def record_hash(rec: dict) -> str:
    """sha256 of one input's record in canonical JSON (tests/test_bench_parity.py
    recomputes it from the device records)."""
    return hashlib.sha256(json.dumps(rec, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def block_hashes(recs):
    out = []
    for b in range(0, len(recs), BLOCK):
        h = hashlib.sha256()
        for r in recs[b:b + BLOCK]:
            h.update(record_hash(r).encode())
        out.append(h.hexdigest()[:32])
    return out


# ---- worker: COMPUTE of one input on the restored post-INIT image ---------------------
_W = {}


def _load(name: str):
    if name.endswith(".man"):
        return rc.load_harness(REPO / "paper_2603_05725_b200" / "workloads" / name)
    return rb.get_benchmark(name).load()


def _winit(name, master_seed):
    m = _load(name)
    image = DeviceMemoryImage(rng=Stream(master_seed, 2000))
    runner = rc.PhaseRunner(m, image)
    assert runner.run_phase(rc.INIT, m.seed(master_seed), iteration=0).status == "ok"
    runner.mark_baseline()
    _W.update(m=m, image=image, runner=runner, snap=image.snapshot())


def _wexec(job):
    it, child = job
    m, image, runner = _W["m"], _W["image"], _W["runner"]
    image.restore(_W["snap"])
    runner.reset_to_baseline()
    delta = CoverageMap.for_program(m.program)
    image._next_alloc_id = PLACEHOLDER
    out = runner.run_phase(rc.COMPUTE, child, coverage=delta, iteration=it)
    return it, out.status, out.retired, image._next_alloc_id - PLACEHOLDER, out.report, delta


# ---- driver --------------------------------------------------------------------------
def campaign(name, *, master_seed, round_size, rounds, keep_prefix, procs):
    """`rounds` = list of input counts per round (a prefix of the last round may be
    given).  Returns per-round dicts."""
    m = _load(name)
    specs = m.argspecs
    seed_tc = m.seed(master_seed)
    corpus = rc.Corpus()
    corpus.add_seed(seed_tc)
    findings = rc.FindingsLog()
    gcov = CoverageMap.for_program(m.program)
    sched = MutationSchedule()
    image = DeviceMemoryImage(rng=Stream(master_seed, 2000))
    runner = rc.PhaseRunner(m, image)
    assert runner.run_phase(rc.INIT, seed_tc, iteration=0).status == "ok"
    next_id = image._next_alloc_id
    out = []
    it0 = 1
    with mp.get_context("fork").Pool(procs, initializer=_winit, initargs=(name, master_seed)) as pool:
        for n in rounds:
            t0 = time.time()
            round_corpus = rc.Corpus(list(corpus.entries))
            jobs, meta = [], []
            for it in range(it0, it0 + n):
                if it == 1:
                    child, pidx = seed_tc, -1
                else:
                    s = Stream(master_seed, KEYBASE + it)
                    parent = rc.schedule_next(round_corpus, s, it)
                    pidx = next(i for i, e in enumerate(round_corpus.entries) if e.tc is parent)
                    child = mutate_testcase(parent, specs, sched, s)
                jobs.append((it, child))
                meta.append(pidx)
            t1 = time.time()
            recs = []
            for k, (it, status, retired, allocs, rep, delta) in enumerate(
                    pool.imap(_wexec, jobs, chunksize=64)):
                child = jobs[k][1]
                fresh = new_edges_since(delta, gcov)
                gcov.merge_from(delta)
                line = None
                if rep is not None:
                    fix = {}
                    for f in ("alloc_id", "provenance"):
                        v = getattr(rep, f)
                        if v is not None and v >= PLACEHOLDER:
                            fix[f] = next_id + (v - PLACEHOLDER)
                    rep = dataclasses.replace(rep, iteration=it, dedupe_key=rep.dedupe_key, **fix)
                    line = rep.to_line()
                    findings.add(rep)
                admitted = rep is None and bool(fresh) and it != 1
                if admitted:
                    corpus.admit(child, it)
                next_id += allocs
                recs.append({"it": it, "parent": meta[k], "child": digest(child), "rng_seed": str(child.rng_seed),
                             "trace": [op.encode() for op in child.trace], "status": status, "retired": retired,
                             "allocs": allocs, "edges": edges_json(delta), "admitted": admitted, "report": line})
            out.append({"it0": it0, "n": n, "blocks": block_hashes(recs), "records": recs[:keep_prefix],
                        "admitted": [r["it"] for r in recs if r["admitted"]],
                        "findings": findings.render_text(), "coverage": report_to_rec(build_report(gcov)),
                        "corpus": [digest(e.tc) for e in corpus.entries], "next_alloc_id": next_id,
                        "int_counts": {str(k): v for k, v in sorted(sched._int_counts.items())}})
            print(f"{name}: round it0={it0} n={n}: mutate {t1 - t0:.1f}s, exec+absorb {time.time() - t1:.1f}s, "
                  f"admitted {len(out[-1]['admitted'])}, findings {len(findings.render_text().splitlines())}",
                  flush=True)
            it0 += n
    return out


C2 = dict(name="matmul.man", master_seed=11, round_size=1 << 20, rounds=[1 << 20, 4096], keep_prefix=20000)
C5 = dict(names=("dot", "amax", "rotm"), master_seed=11, round_size=1 << 14, rounds=[1 << 14, 1 << 14],
          keep_prefix=2000)


def _write(path: Path, obj) -> None:
    with gzip.open(path, "wt", compresslevel=9) as f:
        json.dump(obj, f, sort_keys=True, separators=(",", ":"))


def main():
    which = sys.argv[1:] or ["c2", "c5"]
    procs = int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 8))
    if "c5" in which:
        runs = {}
        for nm in C5["names"]:
            runs[nm] = campaign(nm, master_seed=C5["master_seed"], round_size=C5["round_size"], rounds=C5["rounds"],
                                keep_prefix=C5["keep_prefix"], procs=procs)
        _write(HERE / "ref_bench_c5.json.gz", {"config": {k: v for k, v in C5.items()}, "keybase": KEYBASE,
                                               "block": BLOCK, "runs": runs})
    if "c2" in which:
        run = campaign(C2["name"], master_seed=C2["master_seed"], round_size=C2["round_size"], rounds=C2["rounds"],
                       keep_prefix=C2["keep_prefix"], procs=procs)
        _write(HERE / "ref_bench_c2.json.gz", {"config": C2, "keybase": KEYBASE, "block": BLOCK, "rounds": run})


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
