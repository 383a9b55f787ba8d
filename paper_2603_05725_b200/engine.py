"""Device round driver: batched rounds of the fuzzing inner loop on a GPU.

A *round* is R consecutive fuzz inputs ``it0 .. it0+R-1`` of the batched-round
contract: every input schedules a parent from the corpus as it
stood at the round start, mutates with its own Philox stream, executes its
COMPUTE phase on the post-INIT baseline, and is absorbed in ``it`` order.
All of it runs as stream-ordered kernels from ``libsfg_b200.so``; torch only
holds device memory and provides streams and events.

Round pipelining.  A round's mutation depends on earlier rounds only through
corpus admissions (rotation counts depend on draws only; alloc ids are
applied on the host).  ``run_rounds`` therefore keeps ``depth`` rounds in
flight on separate streams, each mutated from the corpus as of its
submission; rounds are finalized (triaged) strictly in order, and when a
round admits a child or stops the campaign every later in-flight round is
re-submitted (or dropped).  The results are identical to running the rounds
one after another; the long-running inputs of one round (the round time is
bounded below by its longest input) overlap with the bulk of the next ones.
"""

from __future__ import annotations

import ctypes
import os
import time
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .baseline import MemConfig, OutOfSpaceError, build_baseline, record_table
from .coverage import CoverageMap
from .findings import FindingsLog
from .sir import SPACE_ORDER
from .lowering import (CHILD, ENTRY, ST_COUNTER, MAX_KERNELS, OV_CAP0, OV_CHUNK, ctx_edge_hashes, ST_FINDING,
                       ST_LANE_RECS, ST_OUT_OF_SPACE, ST_OVERLAY, ST_ZERO_ALLOC, VAL, VERDICT, Lowered, LoweringError,
                       decode_op, decode_verdict, ov_bytes, pack_values, unpack_values)
from .shard import RoundComm, owner_of
from .testcase import MutationError, TestCase

NONE = 0x7FFFFFFF   # "no index" in the triage MIN buffers (sfg.h)
STATUS = {0: "ok", 1: "finding", 2: "budget"}
DEFAULT_SOFT_CAP = 1 << 15   # retired instructions before an input moves to the tail pass
SEQ_PAR_MIN = 64      # sequential discipline: smaller rounds walk the stream on one thread
SEQ_ROUND0 = 4096     # sequential discipline: first round size (doubles while rounds run to their end)


class CorpusDev(ctypes.Structure):
    _fields_ = [("meta", ctypes.c_void_p), ("vals", ctypes.c_void_p), ("data", ctypes.c_void_p),
                ("n", ctypes.c_int32), ("n_seeds", ctypes.c_int32)]


@dataclass(frozen=True)
class MutationConfig:
    """Mirror of the reference ``MutationConfig`` (mutation.py:389-393)."""
    granule: int = 4
    redzone: int = 32
    max_ops: int = 3


class DeviceFatal(Exception):
    pass


def _ptr(t):
    return None if t is None else t.data_ptr()


def _np(t: torch.Tensor, dtype) -> np.ndarray:
    return t.detach().cpu().numpy().view(dtype)


def _align16(n: int) -> int:
    return (n + 15) // 16 * 16


class RoundResult:
    """Host-side outcome of one finalized round."""

    def __init__(self, it0, n, stop, executed, admitted, new_keys, slot):
        # global round: inputs it0 .. it0+n-1; stop / executed over all ranks
        self.it0, self.n, self.stop, self.executed = it0, n, stop, executed
        self.n_admitted = admitted
        self.new_keys = new_keys          # [(round index, BugReport)] for keys first seen here
        self.slot = slot


_STREAMS: dict = {}


def _round_stream(L, dev, index: int):
    """Process-wide stream of round slot ``index`` (created on first use, reused by
    every campaign of the process): rounds in flight keep distinct hardware queues.
    index < 0: a private torch stream (auxiliary slots)."""
    if index < 0:
        return torch.cuda.Stream(device=dev)
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), index)
    if key not in _STREAMS:
        with torch.cuda.device(key[0]):
            h = ctypes.c_void_p()
            _native.check(L.sfg_stream_create(0, ctypes.byref(h)), "stream")
            _STREAMS[key] = torch.cuda.ExternalStream(h.value, device=torch.device("cuda", key[0]))
    return _STREAMS[key]


class Slot:
    """Device buffers + stream of one in-flight round."""

    def __init__(self, dc: "DeviceCampaign", cap: int, index: int = -1):
        dev = dc.dev
        C, E, A = max(dc.C, 1), max(dc.E, 1), dc.n_args
        i64 = lambda m: torch.empty(max(m, 1), dtype=torch.int64, device=dev)  # noqa: E731
        i32 = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=dev)  # noqa: E731
        u8 = lambda m: torch.empty(max(m, 16), dtype=torch.uint8, device=dev)  # noqa: E731
        self.cap = cap
        self.stream = _round_stream(dc.L, dev, index)
        # the long-input pass runs on a high-priority stream: its CTAs are dispatched
        # ahead of other rounds' bulk CTAs whenever SM slots free up
        self.tail_stream = torch.cuda.Stream(device=dev, priority=-1) if dc.tail_priority else self.stream
        # triage / commit of a finalized round: high priority, so the host's wait for the
        # round's verdict scalars does not queue behind later rounds' bulk CTAs
        self.fin = torch.cuda.Stream(device=dev, priority=-1)
        self.parent, self.picks, self.flags, self.prefix = i32(cap), u8(cap * 3), i32(cap * C), i64(cap * C)
        self.children, self.vals = u8(cap * CHILD.itemsize), u8(cap * A * VAL.itemsize)
        self.work_base, self.ro_base = i64(cap), i64(cap)
        self.verdicts, self.ecnt = u8(cap * VERDICT.itemsize), i32(cap * E)
        self.allocs, self.allocs_prefix, self.admit, self.pos = i64(cap), i64(cap), i64(cap), i64(cap)
        self.bytes, self.boff, self.sel, self.dst_off = i64(cap), i64(cap), i32(cap), i64(cap * A)
        # scan totals: [0..8) layout/admission scans, [8..8+C) rotation-count columns
        self.tmp, self.tot = i64((cap + 2047) // 2048 + 8), i64(8 + 16)
        self.counter = i32(8)            # work counters of this slot's execute launches
        self.deferred = i32(2 * cap)     # tail-pass lists: soft-cap deferrals, sequential re-runs
        self.order = i32(cap)            # bulk-pass schedule (sfg_order)
        self.rep, self.n_live = i32(cap), i32(1)   # duplicate inputs' representatives (sfg_dedupe)
        self.dup_slots = 1 << max(2 * cap - 1, 1).bit_length()
        # allocated with the slot, never mid-pipeline (a cudaMalloc there stalls the device)
        self.dup_table = torch.zeros(self.dup_slots, dtype=torch.int64, device=dev) \
            if (dc.dedupe or dc.group_dups) else None
        self.group_scratch = i32(int(dc.L.sfg_group_scratch_ints(cap))) if dc.group_dups else None
        self.full_order = i32(cap) if dc.group_dups else None   # grouped schedule (sfg_group_schedule)
        # sequential discipline: worker stream state before every input and after the last
        self.states = u8((cap + 1) * dc.state_bytes) if dc.sequential else None
        self.seq_par, self.seq_scratch, self.seq_words = False, None, 0
        self.start_state = u8(dc.state_bytes) if dc.sequential else None
        self.seq_prev = None             # the in-flight round this one continues (pipelined)
        self.fused = False               # the execute pass builds the work regions itself
        self.ev_gen = None               # children generated (the next round may read states[n])
        self.reader_ev = None            # the next round has copied states[n]
        self.seq_stats = i64(2)          # seqgen: [children found, words they drew]
        self.pin_seq = torch.zeros(2, dtype=torch.int64, pin_memory=True)
        self.order_scratch = i32(int(dc.L.sfg_order_scratch_ints(cap)))
        # triage partials (merged across ranks between the phases, sfg.h):
        # MIN: [stop, fatal, first_hit[E], key_first[K]]; SUM: [edge_delta[E], key_count[K], entered[16]]
        E0, K0 = dc.E, dc.K
        self.mins = i32(2 + E0 + K0)
        self.scalars, self.first, self.kfirst = self.mins[:2], self.mins[2:2 + E0], self.mins[2 + E0:2 + E0 + K0]
        self.sums = i64(E0 + K0 + MAX_KERNELS)
        self.edelta, self.kcount, self.ent = self.sums[:E0], self.sums[E0:E0 + K0], self.sums[E0 + K0:]
        self.small = i64(2)              # [admitted, allocs] of this rank, all-gathered
        self.counts_base = torch.zeros(C, dtype=torch.int64, device=dev)
        self.counts_after = torch.zeros(max(C, 1), dtype=torch.int64, device=dev)
        self.pin_ca = torch.zeros(max(C, 1), dtype=torch.int64, pin_memory=True)
        self.counts_after_valid = False
        self.sat_base = False            # counts_base holds the frozen (saturated) counts
        self.sat_round = False           # the round was submitted with saturated counts
        self.pin_tot = torch.empty(8 + 16, dtype=torch.int64, pin_memory=True)
        self.pin_sc = torch.empty(2, dtype=torch.int32, pin_memory=True)
        self.pin_gath = torch.empty((dc.comm.world, 2), dtype=torch.int64, pin_memory=True)
        self.pin_kc = torch.empty(max(K0, 1), dtype=torch.int64, pin_memory=True)
        self.work, self.work_cap = None, 0
        self.readouts = None
        self.ev_counts = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()
        self.exec_ev = None
        self.it0 = self.n = 0            # this rank's slice: global ids it0 .. it0+n-1
        self.round_it0 = self.round_n = 0  # the whole (global) round
        self.i_base = 0                  # round index of this rank's first input
        self.executed = 0                # this rank's inputs at or before the stop
        self.alloc_base = 0              # alloc id of this rank's first allocation
        self.round_index = -1

    def ensure_work(self, nbytes: int, dev):
        if nbytes > self.work_cap:
            self.work_cap = int(nbytes * 1.1) + 4096
            self.work = self.alloc_on_stream(self.work, self.work_cap, dev)

    def alloc_on_stream(self, old, nbytes: int, dev):
        """A new buffer for this slot's stream, replacing ``old``: superseded kernels
        queued on the stream may still use the old one, so it is recorded on the stream
        (the caching allocator reuses it only after that work completes), and the new
        one is allocated in the stream's pool (reuse is stream-ordered)."""
        if old is not None:
            old.record_stream(self.stream)
        with torch.cuda.stream(self.stream):
            return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=dev)


class DeviceCampaign:
    def __init__(self, manifest, *, master_seed=1, mem: MemConfig | None = None,
                 mutation: MutationConfig | None = None, budget=1_000_000, window=256, recent_weight=4.0,
                 diff_readback=False, stop_on_first_finding=False, stop_bug_class=None, device=None,
                 extra_seeds=(), ids_reset_per_input=False, comm: RoundComm | None = None,
                 soft_cap: int | None = None, ctx_map_bits: int = 0, fanout: int = 0, sequential: bool = False,
                 dedupe: bool = False,
                 baseline=None, jit: bool = True, term_phase: bool = False):
        if not torch.cuda.is_available():
            raise _native.NativeError("no CUDA device: the fuzzing inner loop runs only on the GPU")
        self.L = _native.lib()
        self.dev = torch.device(device or "cuda")
        self.comm = comm or RoundComm()
        # sequential: the reference fuzz_loop's own stream discipline (one worker stream,
        # rounds cut after each admission) instead of the batched-round contract
        self.sequential = bool(sequential)
        self.seq_single = os.environ.get("SFG_SEQ_SINGLE", "0") == "1"   # force the one-thread walk (tests / A-B)
        self._seq_mu = 12.0            # words per child (seqgen candidate range), refined per round
        self.seq_scratch = None        # seqgen successor levels + path (one per campaign)
        self._seq_gen_ev = None        # the last submitted generation
        self.seq_truncations = 0
        # K2 fused into the bulk pass (sfg_execute with the corpus); SFG_FUSE_APPLY=0:
        # a separate sfg_apply pass (A/B, tests)
        self.fuse_apply = os.environ.get("SFG_FUSE_APPLY", "1") != "0"
        # opt-in: duplicate inputs of a round executed once (sfg_dedupe; SFG_DEDUPE=1/0
        # overrides for A/B).  Off by default: every input runs.
        self.dedupe = bool(dedupe) if "SFG_DEDUPE" not in os.environ else os.environ["SFG_DEDUPE"] == "1"
        # equal inputs scheduled side by side in the bulk pass (all of them run); SFG_GROUP_DUPS=0: off
        self.group_dups = os.environ.get("SFG_GROUP_DUPS", "1") != "0"
        self.state_bytes = int(self.L.sfg_stream_state_bytes())
        if self.sequential and (self.comm.world > 1 or fanout):
            raise LoweringError("the sequential discipline runs on one device without fan-out")
        if soft_cap is None:
            soft_cap = int(os.environ.get("SFG_SOFT_CAP", DEFAULT_SOFT_CAP))
        self.soft_cap = soft_cap
        # bulk pass in signature order (sfg_order): warps of inputs likely to share a path
        self.order_inputs = os.environ.get("SFG_ORDER", "1") != "0"
        self.tail_priority = os.environ.get("SFG_TAIL_PRIO", "0") != "0"
        self.manifest = manifest
        self.mem = mem or MemConfig()
        self.mutation = mutation or MutationConfig()
        self.master_seed = master_seed
        self.seed_tc = manifest.seed(master_seed)
        self.budget = budget
        # the post-INIT state; INIT launches run on the device (_init_launch)
        self.base = baseline if baseline is not None else build_baseline(manifest, self.seed_tc, self.mem,
                                                                            init_launch=self._init_launch)
        stop_class = None
        if stop_bug_class is not None:
            stop_class = getattr(stop_bug_class, "value", str(stop_bug_class))
        self.low = Lowered(manifest, self.base, mem=self.mem, mutation=self.mutation, master_seed=master_seed,
                           budget=budget, window=window, recent_weight=recent_weight,
                           diff_readback=diff_readback, stop_first=stop_on_first_finding, stop_class=stop_class,
                           fanout=fanout, term_phase=term_phase, jit=jit)
        self.diff = bool(diff_readback)
        self.specs = manifest.argspecs
        self.n_args = len(self.specs)
        self.C = len(self.low.int_args)
        if self.C > 16:     # sfg_prog.int_slot columns (SFG_MAX_ARGS)
            raise LoweringError("more than 16 i32 arguments")
        self.E = self.low.n_edges
        self.K = self.low.n_keys
        recs = record_table(self.base, self.low.labels)
        # padded to whole copy-on-write chunks (a chunk is copied whole on its first write)
        blob = bytearray(self.base.blob)
        blob += bytes(-len(blob) % OV_CHUNK or (OV_CHUNK if not blob else 0))
        self.blob = torch.frombuffer(blob, dtype=torch.uint8).to(self.dev)
        # host<->device bytes moved by the campaign (bench e2e accounting)
        self.h2d_bytes = len(self.base.blob)
        self.d2h_bytes = 0
        h = ctypes.c_void_p()
        P = self.low.prog_bytes()
        _native.check(self.L.sfg_program_create(
            P, len(P), self.low.ins.ctypes.data, len(self.low.ins), self.low.hostops.ctypes.data,
            len(self.low.hostops), self.low.binds.ctypes.data, len(self.low.binds), recs.ctypes.data, len(recs),
            self.low.const_blob, len(self.low.const_blob), self.blob.data_ptr(), ctypes.byref(h)),
            "sfg_program_create")
        self.h = h
        self.h2d_bytes += (len(P) + self.low.ins.nbytes + self.low.hostops.nbytes + self.low.binds.nbytes +
                           recs.nbytes + len(self.low.const_blob))
        self.jit = self.L.sfg_program_jit_source(self.h, None, 0) > 0
        # global campaign state on device
        self.edge_total = torch.zeros(max(self.E, 1), dtype=torch.int64, device=self.dev)
        self.ghit = torch.zeros(max(self.E, 1), dtype=torch.uint8, device=self.dev)
        self.entered = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.counts_run = torch.zeros(max(self.C, 1), dtype=torch.int64, device=self.dev)
        # MutationSchedule rotation counts only steer generation while below 3
        # (mutation.py:378-386): once every mutable int column has reached 3 they are
        # saturated for the rest of the worker, and a round needs neither the plan
        # pass nor the per-column pick scans (sfg_mutate with a NULL prefix)
        P0 = self.low.prog
        self._sat_cols = [int(P0["int_slot"][a]) for a in range(int(P0["n_args"]))
                          if int(P0["int_slot"][a]) >= 0 and not int(P0["arg_fixed"][a])]
        self._counts_sat = not self._sat_cols
        self.seq_state = torch.zeros(self.state_bytes, dtype=torch.uint8, device=self.dev)
        self._set_worker_stream(0)
        # context-sensitive hashed coverage map (derived view, csrc/ctxmap.cu)
        self.ctx_bits = int(ctx_map_bits)
        if self.ctx_bits:
            self.ctx_map = torch.zeros(max(1 << self.ctx_bits, 4), dtype=torch.uint8, device=self.dev)
            self.edge_ctx = torch.from_numpy(ctx_edge_hashes(self.low, manifest).view(np.int64)).to(self.dev)
            self.ctx_new = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.next_alloc_id = self.base.next_id
        self.ids_reset = ids_reset_per_input   # reinit mode: every input gets a fresh image
        self.findings = FindingsLog()
        self.key_strings: dict = {}
        # corpus (device) + host mirror
        self.cap = self.data_cap = self.n_corpus = self.corpus_bytes = 0
        self.max_entry_work = 0
        self.host_entries: list = []     # (TestCase, admitted_iteration, is_seed)
        from .interop import as_testcase
        seeds = [self.seed_tc] + [as_testcase(t) for t in extra_seeds]
        self._upload_seeds(seeds)
        self.n_seeds = len(seeds)
        self.slots: list[Slot] = []
        self._last_done = None           # event: previous round finalized
        self._last_counts = None         # event: counts_run valid for the next submission
        self.rounds = 0
        self.spec_depth = int(os.environ.get("SFG_SPEC0", "2"))   # adaptive speculation depth (run_rounds)
        self.launches = 0                # kernels launched through the C ABI (bench evidence)
        self.ov_grows = 0                # copy-on-write overlay enlargements (rounds re-run)
        self.timing = False              # record CUDA events around each execute kernel
        self.exec_events: list = []
        # stage profiling (bench.py per-kernel rooflines): when a list, every round
        # appends (stage name, CUDA event) marks on its stream at stage boundaries
        self.stage_marks = None
        # diagnostics: host clock of every submission / finalization (SFG_ROUND_LOG=1)
        self.round_log = [] if os.environ.get("SFG_ROUND_LOG") else None

    # ---- INIT launches / TERM phase: one-input device programs ------------------------
    def _phase_program(self, script, baseline, *, term=False):
        """A device program whose COMPUTE script is ``script`` over ``baseline``
        (generic interpreter, no NVRTC: it runs once)."""
        from dataclasses import replace
        from .manifest import COMPUTE, INIT, TERM, HostOp
        allocs = [o for o in self.manifest.phases[INIT] if o.kind == "alloc"]
        allocs += [HostOp("alloc", 0, name=n) for n in baseline.named if n.startswith("\0")]
        m2 = replace(self.manifest, phases={INIT: allocs, COMPUTE: list(script), TERM: []})
        return DeviceCampaign(m2, master_seed=self.master_seed, mem=self.mem, mutation=self.mutation,
                              budget=self.budget, diff_readback=True, device=self.dev, baseline=baseline,
                              jit=False, term_phase=term)

    def _init_launch(self, op, state, live):
        """One INIT launch (build_baseline): run it on the device over the state so
        far and read back the final bytes of every live record (campaign.py:483-561
        with phase INIT: no coverage, the seed input, iteration 0)."""
        from .baseline import InitFailure
        from .manifest import HostOp
        recs = state.records
        outs = [HostOp("copy_out", op.line, name=n, size=recs[state.named[n][2]].size) for n in live]
        dc = self._phase_program([op] + outs, state)
        try:
            (res,) = dc.execute_testcases([self.seed_tc], iteration0=0)
        finally:
            dc.close()
        if res["status"] != "ok":   # campaign.py:723-725
            raise InitFailure(f"init phase failed on the seed input: {res['status']}")
        return {n: res["readouts"][n] for n in live}

    def run_term(self):
        """The TERM phase of a worker (campaign.py:756-762): on the restored post-INIT
        state with the seed input, iteration -1; returns its BugReport or None.
        Allocation ids continue the worker's counter."""
        from .baseline import term_frees_clean
        from .manifest import TERM
        ops = self.manifest.phases[TERM]
        if not ops or term_frees_clean(self.base, ops):
            return None
        dc = self._phase_program(ops, self.base, term=True)
        try:
            (res,) = dc.execute_testcases([self.seed_tc], iteration0=-1, id_base=self.next_alloc_id)
        finally:
            dc.close()
        if res["status"].startswith("fatal"):
            raise DeviceFatal(f"TERM phase: {res['status']}")
        return res["report"]

    # ---- corpus ---------------------------------------------------------------------
    def _u8(self, n):
        return torch.empty(max(int(n), 16), dtype=torch.uint8, device=self.dev)

    def _grow_corpus(self, cap, data_cap):
        cap, data_cap = max(cap, self.cap), max(data_cap, self.data_cap)
        if cap == self.cap and data_cap == self.data_cap:
            return
        torch.cuda.synchronize(self.dev)  # in-flight rounds may still read the old buffers
        meta, vals = self._u8(cap * ENTRY.itemsize), self._u8(cap * self.n_args * VAL.itemsize)
        chld, data = self._u8(cap * CHILD.itemsize), self._u8(data_cap)
        if self.cap:
            for new, old, nb in ((meta, self.c_meta, self.cap * ENTRY.itemsize),
                                 (vals, self.c_vals, self.cap * self.n_args * VAL.itemsize),
                                 (chld, self.c_child, self.cap * CHILD.itemsize), (data, self.c_data, self.data_cap)):
                new[:nb].copy_(old[:nb])
        self.c_meta, self.c_vals, self.c_child, self.c_data = meta, vals, chld, data
        self.cap, self.data_cap = cap, data_cap

    def _entry_work_bound(self, vals) -> int:
        """Upper bound of a child's work-region bytes given its parent's values: the
        array mutations at most double an array (array_dim), or set 4*count
        (array_extreme), so bound each array by max(2*nbytes, 8*count) + 16."""
        b = 0
        mask = int(self.low.prog["copy_src_mask"])
        for a, v in enumerate(vals):
            if v["kind"] == 2:
                ov = int(v["size_override"])
                grow = max(2 * int(v["nbytes"]), 8 * int(v["count"])) + 16
                b += _align16(max(grow, ov if ov != -(1 << 63) else 0))
                if mask >> a & 1:     # pristine copy of a copy_in source
                    b += _align16(grow)
        return b + int(self.low.prog["named_work_bytes"]) + ov_bytes(int(self.low.prog["ov_cap"]))

    def _upload_seeds(self, seeds):
        metas = np.zeros(len(seeds), ENTRY)
        allv, blob = [], bytearray()
        for j, tc in enumerate(seeds):
            vals, payload = pack_values(tc, self.specs)
            vals["data_off"] += np.where(vals["kind"] == 2, len(blob), 0).astype(np.uint64)
            blob += payload
            allv.append(vals)
            metas[j] = (0, tc.rng_seed & ((1 << 64) - 1), 1, -1, 0)
            self.host_entries.append((tc, 0, True))
            self.max_entry_work = max(self.max_entry_work, self._entry_work_bound(vals))
        self._grow_corpus(max(64, len(seeds) * 2), max(1 << 16, len(blob) * 2))
        v = np.concatenate(allv)
        self.c_meta[:metas.nbytes].copy_(torch.frombuffer(bytearray(metas.tobytes()), dtype=torch.uint8))
        self.c_vals[:v.nbytes].copy_(torch.frombuffer(bytearray(v.tobytes()), dtype=torch.uint8))
        if blob:
            self.c_data[:len(blob)].copy_(torch.frombuffer(blob, dtype=torch.uint8))
        self.n_corpus, self.corpus_bytes = len(seeds), len(blob)
        self.h2d_bytes += metas.nbytes + v.nbytes + len(blob)

    def corpus_dev(self) -> CorpusDev:
        return CorpusDev(self.c_meta.data_ptr(), self.c_vals.data_ptr(), self.c_data.data_ptr(),
                         self.n_corpus, self.n_seeds)

    # ---- slots -----------------------------------------------------------------------
    def _slot(self, k: int, n: int) -> Slot:
        while len(self.slots) <= k:
            self.slots.append(None)
        s = self.slots[k]
        if s is None or s.cap < n:
            s = Slot(self, max(n, 1024), k)
            self.slots[k] = s
        return s

    def _scan64(self, S: Slot, src, n, stride, col, out, total_slot, stream=None):
        self.launches += 3
        _native.check(self.L.sfg_scan_u64(src.data_ptr(), n, stride, col, out.data_ptr(), 1, 0, S.tmp.data_ptr(),
                                          S.tot.data_ptr() + 8 * total_slot, (stream or S.stream).cuda_stream),
                      "scan")

    def _set_worker_stream(self, w: int):
        """Worker w's stream Stream(master_seed, 1000 + w) (campaign.py:714)."""
        buf = (ctypes.c_uint8 * self.state_bytes)()
        self.L.sfg_stream_state_init(self.master_seed & ((1 << 64) - 1), 1000 + w, buf)
        self.seq_state.copy_(torch.frombuffer(bytearray(buf), dtype=torch.uint8))

    def new_worker(self, w: int = 0):
        """Reference workers (campaign.py:712-730) get a fresh MutationSchedule and a fresh
        image: rotation counts and alloc ids restart; corpus/findings/coverage are shared.
        Sequential discipline: the worker's own stream too."""
        self.drain()
        self.counts_run.zero_()
        self._last_counts = None
        self._counts_sat = not self._sat_cols
        self.next_alloc_id = self.base.next_id
        if self.sequential:
            self._set_worker_stream(w)

    def drain(self):
        torch.cuda.synchronize(self.dev)

    # ---- submit: mutate + execute (speculative on the current corpus) -----------------
    def _submit(self, S: Slot, it0: int, n: int, round_index: int, resubmit: bool = False):
        """Round ``it0 .. it0+n-1`` (global); this rank mutates and executes its slice."""
        L, hp, comm = self.L, self.h, self.comm
        st = S.stream
        s = st.cuda_stream
        if it0 + n - 1 >= 2 and self.low.prog["n_mutable"] == 0:
            raise MutationError("no mutable arguments")
        lo, hi = comm.bounds(n)
        S.round_it0, S.round_n, S.i_base = it0, n, lo
        S.it0, S.n, S.round_index = it0 + lo, hi - lo, round_index
        it0, n = S.it0, S.n
        cd = self.corpus_dev()
        C = self.C
        if self.sequential:
            self._submit_sequential(S, cd, resubmit)
            return
        if self.timing:
            S.sub_ev = torch.cuda.Event(enable_timing=True)
            S.sub_ev.record(st)
            S.sub_host = time.perf_counter()
        self._mark(S, "submit")
        # a re-submitted round keeps the rotation-count mode it was first submitted in
        # (its base and prefix must not change); a fresh one uses the current mode
        sat = S.sat_round if resubmit else self._counts_sat
        S.sat_round = sat
        if sat:
            # saturated rotation counts: no plan pass, no pick scans; counts_run is
            # frozen (every mutable column >= 3) and serves as every round's base
            self.launches += 1
            prefix = None
            S.counts_after_valid = False
            if not S.sat_base and not resubmit:
                with torch.cuda.stream(st):
                    if self._last_counts is not None:
                        st.wait_event(self._last_counts)
                    S.counts_base.copy_(self.counts_run)
                S.sat_base = True
        else:
            self.launches += 2 + 3 * C
            S.sat_base = False
            prefix = S.prefix.data_ptr()
            _native.check(L.sfg_plan(hp, ctypes.byref(cd), it0, n, S.parent.data_ptr(), S.picks.data_ptr(),
                                     S.flags.data_ptr(), s), "plan")
            for c in range(C):
                _native.check(L.sfg_scan_u32(S.flags.data_ptr(), n, C, c, S.prefix.data_ptr(), C, c,
                                             S.tmp.data_ptr(), S.tot.data_ptr() + 8 * (8 + c), s), "scan flags")
            with torch.cuda.stream(st):
                if not resubmit:                   # a re-submitted round keeps its rotation base
                    if self._last_counts is not None:
                        st.wait_event(self._last_counts)
                    S.counts_base.copy_(self.counts_run)
                    if C:
                        # rotation counts: picks of earlier slices of the round come first
                        g = comm.all_gather(S.tot[8:8 + C], st)
                        S.counts_base[:C] += g[:comm.rank].sum(0)
                        self.counts_run[:C] += g.sum(0)
                    S.counts_after.copy_(self.counts_run)   # read at finalize: saturated yet?
                    S.counts_after_valid = True
                    S.ev_counts.record(st)
                    self._last_counts = S.ev_counts
        _native.check(L.sfg_mutate(hp, ctypes.byref(cd), it0, n, prefix, S.counts_base.data_ptr(),
                                   S.children.data_ptr(), S.vals.data_ptr(), s), "mutate")
        cw = CHILD.itemsize // 8
        self._scan64(S, S.children.view(torch.int64), n, cw, CHILD.fields["work_bytes"][1] // 8, S.work_base, 0)
        S.ensure_work(n * self.max_entry_work + 64, self.dev)
        if self.diff:
            self._scan64(S, S.children.view(torch.int64), n, cw, CHILD.fields["readout_bytes"][1] // 8, S.ro_base, 1)
            with torch.cuda.stream(st):
                S.tot[:2].cpu()  # host needs the readout size (diff mode only; tests)
            S.readouts = S.alloc_on_stream(S.readouts, int(S.tot[1].item()) + 16, self.dev)
        else:
            if S.readouts is not None:
                S.readouts.record_stream(st)
            S.readouts = None
        self._mark(S, "mutated")
        S.fused = self.fuse_apply
        if not S.fused:
            _native.check(L.sfg_apply(hp, ctypes.byref(cd), n, S.children.data_ptr(), S.vals.data_ptr(),
                                      S.work_base.data_ptr(), S.work.data_ptr(), s), "apply")
        self._mark(S, "applied")
        self._execute(S, n, self.soft_cap, cd)

    def _mark(self, S: Slot, name: str, stream=None):
        if self.stage_marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream or S.stream)
            self.stage_marks.append((S.round_index, name, ev))

    def _submit_sequential(self, S: Slot, cd, resubmit: bool = False):
        """Children of the round from the worker stream, one after another (sfg_plan_seq),
        then the same layout scan, payloads and execute as the batched path."""
        L, hp, st = self.L, self.h, S.stream
        s = st.cuda_stream
        it0, n = S.it0, S.n
        if it0 + n - 1 >= 2 and self.low.prog["n_mutable"] == 0:
            raise MutationError("no mutable arguments")
        prev = getattr(S, "seq_prev", None)
        with torch.cuda.stream(st):
            if S.reader_ev is not None:         # the round that started from this slot's end has read it
                st.wait_event(S.reader_ev)
                S.reader_ev = None
            if self._last_done is not None:     # the previous round's cut fixes our start
                st.wait_event(self._last_done)
            if not resubmit:
                # the round's start: the previous round's end state while speculating
                # (pipelined rounds), else the worker state after the last finalized round
                if prev is not None:
                    st.wait_event(prev.ev_gen)
                    sb = self.state_bytes
                    S.start_state.copy_(prev.states[prev.n * sb:(prev.n + 1) * sb])
                    ev = torch.cuda.Event()
                    ev.record(st)
                    prev.reader_ev = ev
                else:
                    S.start_state.copy_(self.seq_state)
            S.counts_base.copy_(self.counts_run)
        # children in parallel (seqgen, sfg_plan_seq_par) when the round's children
        # depend on nothing but the stream: it0 >= 2, saturated rotation counts, no
        # corpus entry leaving the recent window inside the round (the round
        # planner cuts there); otherwise one thread walks the stream
        S.seq_par = it0 >= 2 and self._counts_sat and n >= SEQ_PAR_MIN and not self.seq_single
        if S.seq_par:
            words = int(self._seq_mu * n * 1.06) + 512   # a truncation costs a round cut, not correctness
            need = int(L.sfg_seq_scratch_ints(n, words))
            # one scratch for the campaign: generations are chained in submission
            # order (each waits for the last one submitted, dropped rounds included)
            if self._seq_gen_ev is not None:
                st.wait_event(self._seq_gen_ev)
            if self.seq_scratch is None or self.seq_scratch.numel() < need:
                if self.seq_scratch is not None:
                    self.seq_scratch.record_stream(st)
                self.seq_scratch = torch.empty(need, dtype=torch.int32, device=self.dev)
            S.seq_scratch = self.seq_scratch
            self.launches += 4 + 2 * max(1, n.bit_length())
            _native.check(L.sfg_plan_seq_par(hp, ctypes.byref(cd), it0, n, S.start_state.data_ptr(), words,
                                             S.counts_base.data_ptr(), S.children.data_ptr(), S.vals.data_ptr(),
                                             S.flags.data_ptr(), S.states.data_ptr(), S.seq_scratch.data_ptr(),
                                             S.seq_scratch.numel(), S.seq_stats.data_ptr(), s), "plan_seq_par")
            S.seq_words = words
        else:
            self.launches += 1
            _native.check(L.sfg_plan_seq(hp, ctypes.byref(cd), it0, n, S.start_state.data_ptr(),
                                         S.counts_base.data_ptr(), S.children.data_ptr(), S.vals.data_ptr(),
                                         S.flags.data_ptr(), S.states.data_ptr(), s), "plan_seq")
        S.ev_gen = torch.cuda.Event()
        S.ev_gen.record(st)
        self._seq_gen_ev = S.ev_gen
        cw = CHILD.itemsize // 8
        self._scan64(S, S.children.view(torch.int64), n, cw, CHILD.fields["work_bytes"][1] // 8, S.work_base, 0)
        S.ensure_work(n * self.max_entry_work + 64, self.dev)
        if self.diff:
            self._scan64(S, S.children.view(torch.int64), n, cw, CHILD.fields["readout_bytes"][1] // 8, S.ro_base, 1)
            with torch.cuda.stream(st):
                S.tot[:2].cpu()
            S.readouts = S.alloc_on_stream(S.readouts, int(S.tot[1].item()) + 16, self.dev)
        else:
            if S.readouts is not None:
                S.readouts.record_stream(st)
            S.readouts = None
        S.fused = self.fuse_apply
        if not S.fused:
            _native.check(L.sfg_apply(hp, ctypes.byref(cd), n, S.children.data_ptr(), S.vals.data_ptr(),
                                      S.work_base.data_ptr(), S.work.data_ptr(), s), "apply")
        self._execute(S, n, self.soft_cap, cd)

    def _execute(self, S: Slot, n: int, soft_cap: int = 0, cd=None):
        """K3: bulk pass (long inputs deferred at ``soft_cap`` retired instructions)
        then the tail pass over the deferred inputs; results equal soft_cap = 0."""
        self.launches += 1
        st = S.stream
        if self.timing:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(st)
        # without a corpus (execute_testcases) payloads cannot be re-materialized:
        # no deferral lists -> thread-sequential, no soft cap
        tail = self.jit and cd is not None
        soft = soft_cap if tail else 0
        order = None
        # duplicate inputs run once (sfg_dedupe): campaign rounds on the scheduled
        # bulk pass, not with diff readback (readouts are per input)
        dedupe = tail and self.order_inputs and self.dedupe and not self.diff
        # every input runs, equal inputs side by side in the schedule (sfg_group_schedule)
        group = tail and self.order_inputs and self.group_dups and not dedupe
        if dedupe or group:
            self.launches += 2
            if S.dup_table is None:   # the mode was switched on after the slot was made
                S.dup_table = torch.zeros(S.dup_slots, dtype=torch.int64, device=self.dev)
            _native.check(self.L.sfg_dedupe(self.h, n, S.children.data_ptr(), S.vals.data_ptr(),
                                            S.dup_table.data_ptr(), S.dup_slots, S.rep.data_ptr(), st.cuda_stream),
                          "dedupe")
        if tail and self.order_inputs:
            self.launches += 3
            _native.check(self.L.sfg_order(self.h, n, S.vals.data_ptr(), S.order.data_ptr(),
                                           S.order_scratch.data_ptr(), S.rep.data_ptr() if (dedupe or group) else None,
                                           S.n_live.data_ptr() if (dedupe or group) else None, st.cuda_stream), "order")
            order = S.order.data_ptr()
            if group:
                self.launches += 7
                if S.group_scratch is None:
                    S.group_scratch = torch.empty(int(self.L.sfg_group_scratch_ints(S.cap)), dtype=torch.int32,
                                                  device=self.dev)
                    S.full_order = torch.empty(S.cap, dtype=torch.int32, device=self.dev)
                _native.check(self.L.sfg_group_schedule(self.h, n, S.rep.data_ptr(), S.order.data_ptr(),
                                                        S.n_live.data_ptr(), S.full_order.data_ptr(),
                                                        S.group_scratch.data_ptr(), st.cuda_stream), "group")
                order = S.full_order.data_ptr()
            self._mark(S, "ordered")
        # the bulk pass builds each input's arrays from its parent itself (sfg_apply
        # fused) when the round has a corpus and nothing was materialized before
        fuse = cd if (cd is not None and S.fused) else None
        _native.check(self.L.sfg_execute(
            self.h, ctypes.byref(fuse) if fuse is not None else None, n, S.children.data_ptr(), S.vals.data_ptr(), S.work_base.data_ptr(), S.work.data_ptr(),
            S.verdicts.data_ptr(), S.ecnt.data_ptr(), _ptr(S.readouts), S.ro_base.data_ptr(),
            S.counter.data_ptr(), soft, S.deferred.data_ptr() if tail else None, self.max_entry_work, order,
            S.n_live.data_ptr() if dedupe else None, st.cuda_stream), "execute")
        if tail:
            self._mark(S, "bulk")
            if self.timing:
                evb = torch.cuda.Event(enable_timing=True)
                evb.record(st)
                S.bulk_ev = evb
            self.launches += 4   # two passes: re-materialize + tail kernel each
            ts = S.tail_stream
            if ts is not st:
                ts.wait_stream(st)
            _native.check(self.L.sfg_execute_deferred(
                self.h, ctypes.byref(cd), n, S.children.data_ptr(), S.vals.data_ptr(), S.work_base.data_ptr(),
                S.work.data_ptr(), S.verdicts.data_ptr(), S.ecnt.data_ptr(), _ptr(S.readouts),
                S.ro_base.data_ptr(), S.counter.data_ptr(), S.deferred.data_ptr(),
                self.max_entry_work, ts.cuda_stream), "execute_deferred")
            if ts is not st:
                st.wait_stream(ts)
            if dedupe:
                self.launches += 1
                _native.check(self.L.sfg_dup_fill(self.h, n, S.rep.data_ptr(), S.verdicts.data_ptr(),
                                                  S.ecnt.data_ptr(), st.cuda_stream), "dup_fill")
            self._mark(S, "tail")
        if self.timing:
            ev[1].record(st)
            S.exec_ev = ev
            # (execute start, bulk pass end, tail passes end) of this round
            self.exec_events.append((ev[0], getattr(S, "bulk_ev", None) if tail else None, ev[1]))

    # ---- finalize: triage in order ------------------------------------------------------
    def _triage_pass(self, S: Slot, cut=None):
        """stop -> [MIN] -> absorb -> [MIN, SUM] -> admit -> scans -> [gather], read
        back to the host.  cut: round index after which inputs are discarded (the
        sequential discipline's cut after an admission), applied as a stop."""
        L, hp, st, comm = self.L, self.h, S.fin, self.comm
        s = st.cuda_stream
        st.wait_stream(S.stream)      # the round's execute (and tail) passes
        n, ib = S.n, S.i_base
        self.launches += 7
        self._mark(S, "triage_start", st)
        with torch.cuda.stream(st):
            S.mins.fill_(NONE)
            S.sums.zero_()
        vp, ep = S.verdicts.data_ptr(), S.ecnt.data_ptr()
        _native.check(L.sfg_triage_stop(hp, n, ib, vp, S.scalars.data_ptr(), s), "triage_stop")
        comm.all_reduce(S.scalars, "min", st)
        if cut is not None:
            with torch.cuda.stream(st):
                S.scalars[:1].clamp_(max=cut)
        _native.check(L.sfg_triage_absorb(hp, n, ib, vp, ep, S.scalars.data_ptr(), S.first.data_ptr(),
                                          S.edelta.data_ptr(), S.kfirst.data_ptr(), S.kcount.data_ptr(),
                                          S.ent.data_ptr(), S.allocs.data_ptr(), s), "triage_absorb")
        comm.all_reduce(S.mins[2:], "min", st)
        comm.all_reduce(S.sums, "sum", st)
        _native.check(L.sfg_triage_admit(hp, n, ib, vp, ep, S.children.data_ptr(), S.scalars.data_ptr(),
                                         S.first.data_ptr(), self.ghit.data_ptr(), S.admit.data_ptr(), s),
                      "triage_admit")
        self._scan64(S, S.admit, n, 1, 0, S.pos, 2, st)
        self._scan64(S, S.allocs, n, 1, 0, S.allocs_prefix, 3, st)
        self._mark(S, "triaged", st)
        with torch.cuda.stream(st):
            S.small.copy_(S.tot[2:4])
            gath = comm.all_gather(S.small, st)
            S.pin_sc.copy_(S.scalars, non_blocking=True)
            S.pin_tot.copy_(S.tot, non_blocking=True)
            S.pin_gath.copy_(gath, non_blocking=True)
            if self.K:
                S.pin_kc[:self.K].copy_(S.kcount, non_blocking=True)
            if S.counts_after_valid and not self._counts_sat:
                S.pin_ca.copy_(S.counts_after, non_blocking=True)
            if self.sequential and S.seq_par:
                S.pin_seq.copy_(S.seq_stats, non_blocking=True)
            self.d2h_bytes += S.pin_sc.nbytes + S.pin_tot.nbytes + S.pin_gath.nbytes + 8 * self.K
            ev = torch.cuda.Event()
            ev.record(st)
        ev.synchronize()
        stop, fatal = (int(x) for x in S.pin_sc.numpy())
        if S.counts_after_valid and not self._counts_sat:
            ca = S.pin_ca.numpy()
            self._counts_sat = all(int(ca[c]) >= 3 for c in self._sat_cols)
        return stop, fatal, S.pin_gath.numpy().copy()

    def _finalize(self, S: Slot) -> RoundResult:
        """Triage one round (sfg.h): the triage pass, then corpus append, map commit,
        findings.  Sequential discipline: a round whose first admission is not its
        last executed input is triaged again, cut right after that admission (the
        later inputs were generated from the pre-admission corpus)."""
        L, hp, st, comm = self.L, self.h, S.fin, self.comm
        s = st.cuda_stream
        ib = S.i_base
        with torch.cuda.stream(st):
            if self._last_done is not None:
                st.wait_event(self._last_done)
        stop, fatal, gathered = self._triage_pass(S)
        # an input that overflowed its copy-on-write overlay: grow the overlay and run
        # the round again (deterministic, so the results are those of a large overlay)
        while fatal != NONE and fatal <= stop and self._fatal_status(S, fatal)[0] == ST_OVERLAY:
            self._grow_overlay()
            S.stream.wait_stream(S.fin)
            self._submit(S, S.round_it0, S.round_n, S.round_index, resubmit=True)
            stop, fatal, gathered = self._triage_pass(S)
        N = S.round_n
        cut = None
        if self.sequential and S.seq_par:
            found, used = (int(x) for x in S.pin_seq.numpy())
            if found > 0:   # words per child, for the next round's candidate range
                self._seq_mu = max(2.0, 0.5 * self._seq_mu + 0.5 * used / found)
            if found < N:
                # the seqgen path ran out of candidates at `found`: the round ends
                # there (states[found] is exact) and the next resumes from it
                if used >= 0.8 * S.seq_words or found == 0:
                    self._seq_mu *= 1.5
                self.seq_truncations += 1
                cut = max(found, 1) - 1
                stop, fatal, gathered = self._triage_pass(S, cut=cut)
        if self.sequential and int(gathered[:, 0].sum()):
            executed0 = N if stop == NONE else stop + 1
            adm = _np(S.admit[:S.n], np.int64)
            first = int(np.argmax(adm != 0))
            if first < executed0 - 1 and (cut is None or first < cut):
                cut = first
                stop, fatal, gathered = self._triage_pass(S, cut=cut)
        if fatal != NONE and fatal <= stop:
            self._raise_fatal(S, fatal)
        executed = N if stop == NONE else stop + 1
        if cut is not None and stop == cut:
            stop = NONE        # a cut is not a campaign stop
        S.executed = max(0, min(S.n, executed - ib))
        if self.ctx_bits:
            self.launches += 1
            _native.check(L.sfg_ctxmap(S.n, self.E, ib, S.ecnt.data_ptr(), S.scalars.data_ptr(),
                                       self.edge_ctx.data_ptr(), self.ctx_map.data_ptr(), self.ctx_bits,
                                       self.ctx_new.data_ptr(), s), "ctxmap")
            comm.all_reduce(self.ctx_map, "max", st)
        n_adm = int(gathered[:, 0].sum())
        self._round_id0 = self.next_alloc_id
        S.alloc_base = self.next_alloc_id + int(gathered[:comm.rank, 1].sum())
        if n_adm:
            self._admit(S, gathered[:, 0])
        _native.check(L.sfg_commit(hp, S.edelta.data_ptr(), S.ent.data_ptr(), self.edge_total.data_ptr(),
                                   self.ghit.data_ptr(), self.entered.data_ptr(), s), "commit")
        new_keys = self._absorb_findings(S)
        self.next_alloc_id += int(gathered[:, 1].sum())
        if self.sequential:
            # the worker stream and the rotation counts resume after the last kept input
            k = S.executed
            with torch.cuda.stream(st):
                self.seq_state.copy_(S.states[k * self.state_bytes:(k + 1) * self.state_bytes])
                if self.C and k:
                    self.counts_run[:self.C] += S.flags[:k * self.C].view(k, self.C).sum(0).to(torch.int64)
            if not self._counts_sat and self._sat_cols:
                with torch.cuda.stream(st):
                    ca = self.counts_run.cpu().numpy()
                self._counts_sat = all(int(ca[c]) >= 3 for c in self._sat_cols)
        S.ev_done.record(st)
        self._last_done = S.ev_done
        S.stream.wait_stream(st)      # the slot's next round starts after its finalize work
        self.rounds += 1
        return RoundResult(S.round_it0, N, None if stop == NONE else stop, executed, n_adm, new_keys, S)

    def _fatal_status(self, S: Slot, g):
        """(status, space, alloc_size, alloc_base) of the first fatal input (global
        round index g), read by its owner and shared with every rank."""
        st = None
        if S.i_base <= g < S.i_base + S.n:
            i = g - S.i_base
            v = _np(S.verdicts[i * VERDICT.itemsize:(i + 1) * VERDICT.itemsize], VERDICT)[0]
            st = (int(v["status"]), int(v["space"]), int(v["alloc_size"]), int(v["alloc_base"]))
        if self.comm.world > 1:
            st = next(x for x in self.comm.all_gather_object(st) if x is not None)
        return st

    def _grow_overlay(self):
        """Double the per-input copy-on-write overlay (sfg_prog.ov_cap)."""
        old = int(self.low.prog["ov_cap"])
        new = max(2 * old, OV_CAP0)
        self.low.prog["ov_cap"] = new
        P = self.low.prog_bytes()
        _native.check(self.L.sfg_program_update(self.h, P, len(P)), "sfg_program_update")
        self.max_entry_work += ov_bytes(new) - ov_bytes(old)
        self.ov_grows += 1

    def _raise_fatal(self, S: Slot, g):
        """The first fatal input (global round index g) raises the reference's
        exception on every rank; its owner reads the status."""
        st, space, need, remain = self._fatal_status(S, g)
        if st == ST_OUT_OF_SPACE:   # the reference's message (device_memory.py:428-430)
            raise OutOfSpaceError(f"{SPACE_ORDER[space].value} scope 0: need {need} bytes, {remain} remain")
        if st == ST_ZERO_ALLOC:
            raise ValueError("allocation size must be positive")
        raise DeviceFatal({ST_LANE_RECS: "per-input allocation table overflow",
                           ST_OVERLAY: "per-input INIT-buffer write overlay overflow",
                           ST_COUNTER: "per-input edge counter overflow"}.get(st, f"status {st}"))

    def _admit(self, S: Slot, per_rank):
        """Append the round's admitted children (all ranks, in id order) to the
        corpus: each rank stages its own rows, the rows are all-gathered, and
        every rank regenerates the payloads from (parent, ops) on its device."""
        L, hp, st, comm = self.L, self.h, S.fin, self.comm
        s = st.cuda_stream
        A = self.n_args
        CB, VB = CHILD.itemsize, A * VAL.itemsize
        mine = int(per_rank[comm.rank])
        T = int(per_rank.sum())
        mx = int(per_rank.max())
        self.launches += 1
        with torch.cuda.stream(st):   # temporaries in the slot stream's pool: reuse is stream-ordered
            return self._admit_on_stream(S, per_rank, A, CB, VB, mine, T, mx)

    def _admit_on_stream(self, S, per_rank, A, CB, VB, mine, T, mx):
        L, hp, st, comm = self.L, self.h, S.fin, self.comm
        s = st.cuda_stream
        stage = self._u8(max(mx, 1) * (CB + VB))
        _native.check(L.sfg_select(hp, S.children.data_ptr(), S.vals.data_ptr(), S.admit.data_ptr(),
                                   S.pos.data_ptr(), S.n, stage.data_ptr(), stage.data_ptr() + max(mx, 1) * CB, s),
                      "select")
        with torch.cuda.stream(st):
            if comm.world > 1:
                g = comm.all_gather(stage[:max(mx, 1) * (CB + VB)], st)
                off = max(mx, 1) * CB
                gch = torch.cat([g[r, :int(c) * CB] for r, c in enumerate(per_rank)])
                gva = torch.cat([g[r, off:off + int(c) * VB] for r, c in enumerate(per_rank)])
            else:
                gch, gva = stage[:mine * CB], stage[max(mx, 1) * CB:max(mx, 1) * CB + mine * VB]
            gch, gva = gch.contiguous(), gva.contiguous()
        nb = self._u8(T * 8)
        boff = torch.empty(max(T, 1), dtype=torch.int64, device=self.dev)
        self.launches += 1
        _native.check(L.sfg_child_bytes(hp, gva.data_ptr(), None, T, nb.data_ptr(), s), "child_bytes")
        self._scan64(S, nb.view(torch.int64), T, 1, 0, boff, 4, st)
        with torch.cuda.stream(st):
            nbytes = int(S.tot[4].item())
        self._grow_corpus(max(self.cap, (self.n_corpus + T) * 2),
                          max(self.data_cap, (self.corpus_bytes + nbytes) * 2))
        cd = self.corpus_dev()
        sel = torch.empty(max(T, 1), dtype=torch.int32, device=self.dev)
        dst_off = torch.empty(max(T, 1) * A, dtype=torch.int64, device=self.dev)
        self.launches += 2
        _native.check(L.sfg_compact(hp, gch.data_ptr(), gva.data_ptr(), None, None, boff.data_ptr(), T,
                                    self.n_corpus, self.corpus_bytes, self.c_meta.data_ptr(), self.c_vals.data_ptr(),
                                    self.c_child.data_ptr(), sel.data_ptr(), dst_off.data_ptr(), s), "compact")
        _native.check(L.sfg_regen(hp, ctypes.byref(cd), T, sel.data_ptr(), gch.data_ptr(), gva.data_ptr(),
                                  dst_off.data_ptr(), self.c_data.data_ptr(), s), "regen")
        first = self.n_corpus
        self.n_corpus += T
        self.corpus_bytes += nbytes
        with torch.cuda.stream(st):
            self._mirror_entries(first, self.n_corpus)
    def _mirror_entries(self, lo, hi):
        """Build reference TestCase objects for corpus entries [lo, hi)."""
        meta = _np(self.c_meta[lo * ENTRY.itemsize:hi * ENTRY.itemsize], ENTRY)
        vals = _np(self.c_vals[lo * self.n_args * VAL.itemsize:hi * self.n_args * VAL.itemsize], VAL)
        chld = _np(self.c_child[lo * CHILD.itemsize:hi * CHILD.itemsize], CHILD)
        offs = [int(v["data_off"]) for v in vals if v["kind"] == 2]
        base = min(offs) if offs else 0
        top = max([int(v["data_off"]) + int(v["nbytes"]) for v in vals if v["kind"] == 2] + [base])
        data = self.c_data[base:top].cpu().numpy().tobytes() if top > base else b""
        self.d2h_bytes += meta.nbytes + vals.nbytes + chld.nbytes + len(data)
        for j in range(hi - lo):
            row = vals[j * self.n_args:(j + 1) * self.n_args]
            args = unpack_values(row, data, base)
            parent_tc = self.host_entries[int(meta[j]["parent"])][0]
            ops = tuple(decode_op(chld[j]["ops"][k]) for k in range(int(chld[j]["n_ops"])))
            self.host_entries.append((TestCase(args, int(meta[j]["rng_seed"]), parent_tc.id, ops),
                                      int(meta[j]["admitted_iteration"]), False))
            self.max_entry_work = max(self.max_entry_work, self._entry_work_bound(row))

    def _id_base(self, S: Slot, prefix: int) -> int:
        return self.base.next_id if self.ids_reset else S.alloc_base + prefix

    def _absorb_findings(self, S: Slot):
        """FindingsLog updates of a round: hit counts of known keys; new keys are
        decoded by the rank owning their first input and shared with all ranks."""
        comm = self.comm
        with torch.cuda.stream(S.fin):
            kc = S.pin_kc.numpy()[:self.K]   # copied with the round's scalars (_finalize)
            hot = np.nonzero(kc)[0]
            if not len(hot):
                return []
            kf = S.kfirst.cpu().numpy()
            self.d2h_bytes += kf.nbytes
            fresh = []
            for k in hot:
                ks = self.key_strings.get(int(k))
                if ks is not None and ks in self.findings:
                    self.findings.bump(ks, int(kc[k]))
                else:
                    fresh.append((int(kf[k]), int(k)))
            fresh.sort()
            mine = [(g, k) for g, k in fresh if S.i_base <= g < S.i_base + S.n]
            reps = []
            if mine:
                idx = torch.tensor([g - S.i_base for g, _ in mine], dtype=torch.long, device=self.dev)
                vt = _np(S.verdicts.view(-1, VERDICT.itemsize)[idx].reshape(-1), VERDICT)
                ap = S.allocs_prefix[idx].cpu().numpy()
                self.d2h_bytes += vt.nbytes + ap.nbytes
                for j, (g, k) in enumerate(mine):
                    reps.append((g, k, decode_verdict(vt[j], self.low, S.round_it0 + g,
                                                      self._id_base(S, int(ap[j])))))
            if comm.world > 1:
                reps = sorted(r for part in comm.all_gather_object(reps) for r in part)
            out = []
            for g, k, rep in reps:
                self.key_strings[k] = rep.dedupe_key
                self.findings.add_many(rep, int(kc[k]))
                out.append((g, rep))
            return out

    # ---- public round API --------------------------------------------------------------
    def _run_rounds_sequential(self, it0, it_stop, round_size, on_round, should_continue, depth=8):
        """Sequential discipline: rounds in worker-stream order, each starting right
        after the previous round's last kept input.  Once the rotation counts are
        saturated, later rounds are submitted speculatively from the end state of the
        round before them (seqgen chains on the device); a round that is cut (an
        admission, or a seqgen truncation) or that admits drops the rounds in flight,
        which are generated again from the cut.  Rounds grow while they run to their
        end and shrink when cut."""
        results = []
        inflight = deque()
        it = it0
        size = min(round_size, SEQ_ROUND0)
        window = int(self.low.prog["window"])
        self.reserve(1, min(round_size, max(it_stop - it0, 1)))
        spec = 1
        prev = None
        k = 0

        def plan(at):
            n = min(size, it_stop - at)
            # a round never spans a corpus entry leaving the recent window
            # (schedule_next's weights change there, campaign.py:593-603)
            flips = [adm + window + 1 for _, adm, seed in self.host_entries if not seed and adm + window + 1 > at]
            return max(1, min(n, min(flips) - at)) if flips else n

        while True:
            while len(inflight) < (spec if self._counts_sat else 1) and it < it_stop and \
                    (should_continue is None or should_continue()):
                n = plan(it)
                S = self._slot(k % max(depth, 1), n)
                k += 1
                S.seq_prev = prev
                self._submit(S, it, n, self.rounds + len(inflight))
                inflight.append(S)
                prev = S
                it += n
                if spec > 1:       # speculating after a clean round: the next one twice as large
                    size = min(round_size, 2 * size)
            if not inflight:
                break
            S = inflight.popleft()
            res = self._finalize(S)
            results.append(res)
            if on_round is not None:
                on_round(res)
            if res.stop is not None:
                self.drain()
                break
            if res.executed < S.round_n or res.n_admitted:
                # the rounds in flight continued past a cut or from the pre-admission
                # corpus: generate them again from the worker state
                inflight.clear()
                prev = None
                it = S.round_it0 + res.executed
                spec = 1
                size = max(SEQ_ROUND0, size // 2) if res.executed < S.round_n else size
            else:
                spec = min(2 * spec, max(depth, 1))
                size = min(round_size, 2 * size)
        return results

    def seq_generate(self, it0: int, n: int, parallel: bool, words: int | None = None):
        """Sequential discipline, generation only (tests / diagnostics): children
        it0 .. it0+n-1 from the current worker state, by the one-thread walk or
        by seqgen.  Returns host copies (children, vals, int flags, states[n + 1],
        stats or None); the worker state is not advanced."""
        self.drain()                     # the worker state of the last finalized round is in place
        S = Slot(self, max(n, 1024), 99)
        cd = self.corpus_dev()
        s = S.stream.cuda_stream
        L, hp = self.L, self.h
        with torch.cuda.stream(S.stream):
            S.stream.wait_stream(torch.cuda.current_stream())
            S.counts_base.copy_(self.counts_run)
        stats = None
        if parallel:
            words = words or int(self._seq_mu * n * 1.25) + 256
            scratch = torch.empty(int(L.sfg_seq_scratch_ints(n, words)), dtype=torch.int32, device=self.dev)
            _native.check(L.sfg_plan_seq_par(hp, ctypes.byref(cd), it0, n, self.seq_state.data_ptr(), words,
                                             S.counts_base.data_ptr(), S.children.data_ptr(), S.vals.data_ptr(),
                                             S.flags.data_ptr(), S.states.data_ptr(), scratch.data_ptr(),
                                             scratch.numel(), S.seq_stats.data_ptr(), s), "plan_seq_par")
        else:
            _native.check(L.sfg_plan_seq(hp, ctypes.byref(cd), it0, n, self.seq_state.data_ptr(),
                                         S.counts_base.data_ptr(), S.children.data_ptr(), S.vals.data_ptr(),
                                         S.flags.data_ptr(), S.states.data_ptr(), s), "plan_seq")
        S.stream.synchronize()
        out = (S.children[:n * CHILD.itemsize].cpu().numpy(), S.vals[:n * self.n_args * VAL.itemsize].cpu().numpy(),
               S.flags[:n * self.C].cpu().numpy(), S.states[:(n + 1) * self.state_bytes].cpu().numpy(),
               S.seq_stats.cpu().numpy() if parallel else None)
        return out

    def reserve(self, depth: int, round_size: int) -> None:
        """Allocate the device buffers of ``depth`` rounds of ``round_size`` inputs
        (and their work arenas for the current corpus) ahead of a pipelined run."""
        for k in range(depth):
            S = self._slot(k, round_size)
            S.ensure_work(round_size * self.max_entry_work + 64, self.dev)

    def run_round(self, it0: int, n: int) -> RoundResult:
        """Submit and finalize one round (no pipelining)."""
        S = self._slot(0, n)
        self._submit(S, it0, n, self.rounds)
        return self._finalize(S)

    def run_rounds(self, it0: int, it_stop: int, round_size: int, depth: int = 8, on_round=None,
                   should_continue=None):
        """Rounds covering iterations [it0, it_stop) with up to ``depth`` rounds in
        flight.  ``on_round(result)`` runs after each round is finalized (before its
        slot is reused).  ``should_continue()`` is asked before every new submission
        (e.g. a wall-clock limit); once it says no, the rounds already in flight are
        finalized and nothing more is submitted.  The pipeline stays full across the
        whole range, so a long campaign is one call.  Returns the list of RoundResults
        (stops early on a stop)."""
        if self.sequential:
            return self._run_rounds_sequential(it0, it_stop, round_size, on_round, should_continue, depth)
        plan = []
        it = it0
        while it < it_stop:
            n = min(round_size, it_stop - it)
            plan.append((it, n))
            it += n
        results = []
        inflight = deque()
        base_round = self.rounds
        nxt = 0

        # every slot this call will use exists before the first submission: allocating
        # device memory mid-pipeline can stall the device behind in-flight rounds
        if plan:
            if self.round_log is not None:
                self.round_log.append(("reserve", -1, time.perf_counter()))
            self.reserve(min(depth, len(plan)), max(n for _, n in plan))
            if self.round_log is not None:
                self.round_log.append(("reserved", -1, time.perf_counter()))

        def submit(k):
            it_k, n_k = plan[k]
            S = self._slot(k % depth, n_k)
            if self.round_log is not None:
                self.round_log.append(("submit", k, time.perf_counter()))
            self._submit(S, it_k, n_k, base_round + k)
            inflight.append((k, S))

        def more():
            return nxt < len(plan) and (should_continue is None or should_continue())

        # Speculation depth adapts: an admission invalidates every round in flight, and
        # admissions cluster at the start of a campaign (new coverage), so the depth
        # drops to 2 after an admitting round and quadruples after each clean one
        # (2 -> 8 -> 32: a campaign's pipeline is full after two clean rounds).
        def fill():
            nonlocal nxt
            while len(inflight) < min(depth, self.spec_depth) and more():
                submit(nxt)
                nxt += 1

        fill()
        while inflight:
            k, S = inflight.popleft()
            if self.round_log is not None:
                self.round_log.append(("finalize", k, time.perf_counter()))
            res = self._finalize(S)
            if self.round_log is not None:
                self.round_log.append(("finalized", k, time.perf_counter()))
            results.append(res)
            if on_round is not None:
                on_round(res)
            if res.stop is not None:
                self.drain()
                break
            if res.n_admitted:
                # later in-flight rounds were mutated from the pre-admission corpus: redo them
                self.spec_depth = 2
                redo = list(inflight)
                inflight.clear()
                for kk, SS in redo:
                    self._submit(SS, SS.round_it0, SS.round_n, SS.round_index, resubmit=True)
                    inflight.append((kk, SS))
            else:
                self.spec_depth = min(4 * self.spec_depth, 1 << 20)
            fill()
        return results

    # ---- bench / e2e helpers ------------------------------------------------------------
    def corpus_host_pinned(self):
        """Pinned host copies of the device corpus (meta, vals, child records, payload)."""
        out = []
        for t, nb in ((self.c_meta, self.n_corpus * ENTRY.itemsize),
                      (self.c_vals, self.n_corpus * self.n_args * VAL.itemsize),
                      (self.c_child, self.n_corpus * CHILD.itemsize), (self.c_data, self.corpus_bytes)):
            h = torch.empty(max(nb, 1), dtype=torch.uint8, pin_memory=True)
            h[:nb].copy_(t[:nb])
            out.append(h)
        return out

    def load_corpus_from_host(self, host, stream=None):
        """Re-upload the corpus from pinned host buffers (stream-ordered H2D copies)."""
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            for t, h in zip((self.c_meta, self.c_vals, self.c_child, self.c_data), host):
                t[:h.numel()].copy_(h, non_blocking=True)

    def algorithmic_exec_bytes(self) -> int:
        """Unavoidable off-chip bytes of one exec in the execute kernel: the child's
        argument payload read once, its 64-byte verdict and a 4*ceil(E/32)-byte
        edge-hit bitmap written."""
        seed = self.host_entries[0][0]
        payload = sum(len(v.data) if hasattr(v, "data") else 4 for v in seed.args)
        return payload + 64 + 4 * ((self.E + 31) // 32)

    def retired_mean(self, S: Slot | None = None) -> float:
        S = S or self.slots[0]
        v = _np(S.verdicts[:S.n * VERDICT.itemsize], VERDICT)
        return float(v["retired"].astype(np.float64).mean())

    # ---- views for tests / reporting ----------------------------------------------------
    def ctx_map_slots(self) -> np.ndarray:
        """Set slots of the context-sensitive hashed map (sorted indices)."""
        self.drain()
        return torch.nonzero(self.ctx_map).flatten().cpu().numpy()

    def coverage_map(self) -> CoverageMap:
        self.drain()
        cov = CoverageMap.for_program(self.manifest.program)
        tot = self.edge_total[:self.E].cpu().numpy().view(np.uint64) if self.E else []
        for e, c in enumerate(tot):
            if c:
                name, edge = self.low.edge_names[e]
                cov.edge_counts[name][edge] = int(c)
        ent = int(self.entered.item()) & 0xFFFFFFFF
        for kidx, name in enumerate(self.low.kernel_names):
            if ent >> kidx & 1:
                cov.entered[name] = True
        return cov

    def _edges_row(self, row):
        edges = {}
        for e in np.nonzero(row[:self.E])[0]:
            name, (a, b) = self.low.edge_names[e]
            edges.setdefault(name, []).append([a, b, int(row[e])])
        return {k: sorted(x) for k, x in edges.items()}

    def round_records(self, res: RoundResult):
        """Per-input records of a finalized round (same shape as oracle.loop records)."""
        S = res.slot
        n = S.executed                    # this rank's inputs up to the stop
        self.drain()
        chld = _np(S.children[:n * CHILD.itemsize], CHILD)
        verd = _np(S.verdicts[:n * VERDICT.itemsize], VERDICT)
        E1 = max(self.E, 1)
        ecnt = S.ecnt[:n * E1].cpu().numpy().view(np.uint32).reshape(n, E1)
        admit = S.admit[:n].cpu().numpy()
        aprefix = S.allocs_prefix[:n].cpu().numpy()
        tcs = self.child_testcases(list(range(n)), S)
        recs = []
        for i in range(n):
            c, v = chld[i], verd[i]
            st = int(v["status"])
            rep = decode_verdict(v, self.low, int(c["it"]), self._id_base(S, int(aprefix[i]))) if st == ST_FINDING else None
            recs.append({"it": int(c["it"]), "parent": int(c["parent"]), "child": tcs[i],
                         "status": STATUS.get(st, f"fatal{st}"), "retired": int(v["retired"]),
                         "allocs": int(v["allocs"]), "edges": self._edges_row(ecnt[i]),
                         "report": rep.to_line() if rep else None, "admitted": bool(admit[i])})
        return recs

    def child_testcases(self, idx, S: Slot | None = None):
        """Reference TestCase objects for round inputs ``idx``: payloads regenerated
        on the device from (parent, ops) with the product kernel, then decoded."""
        S = S or self.slots[0]
        n = len(idx)
        if n == 0:
            return []
        st = S.stream
        sel = torch.tensor(list(idx), dtype=torch.int32, device=self.dev)
        with torch.cuda.stream(st):
            vals = _np(S.vals.view(-1, VAL.itemsize * self.n_args)[sel.long()].reshape(-1), VAL)
            chld = _np(S.children.view(-1, CHILD.itemsize)[sel.long()].reshape(-1), CHILD)
        offs = np.zeros(n * self.n_args, np.uint64)
        cur = 0
        for j in range(n):
            for a in range(self.n_args):
                v = vals[j * self.n_args + a]
                if v["kind"] == 2:
                    offs[j * self.n_args + a] = cur
                    cur += _align16(int(v["nbytes"]))
        dst = self._u8(cur + 16)
        doff = torch.from_numpy(offs.view(np.int64)).to(self.dev)
        cd = self.corpus_dev()
        self.launches += 1
        torch.cuda.synchronize(self.dev)
        _native.check(self.L.sfg_regen(self.h, ctypes.byref(cd), n, sel.data_ptr(), S.children.data_ptr(),
                                       S.vals.data_ptr(), doff.data_ptr(), dst.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "regen")
        data = dst.cpu().numpy().tobytes()
        out = []
        for j in range(n):
            row = vals[j * self.n_args:(j + 1) * self.n_args].copy()
            for a in range(self.n_args):
                if row[a]["kind"] == 2:
                    row[a]["data_off"] = offs[j * self.n_args + a]
            c = chld[j]
            p = int(c["parent"])
            if p < 0:
                out.append(self.seed_tc)
                continue
            out.append(TestCase(unpack_values(row, data), int(c["rng_seed"]), self.host_entries[p][0].id,
                                tuple(decode_op(c["ops"][k]) for k in range(int(c["n_ops"])))))
        return out

    # ---- one-shot execution of given test cases (execute_once analogue) -------------------
    def execute_testcases(self, tcs, iteration0: int = 0, trace: bool = False, trace_cap: int = 1 << 16,
                          id_base: int | None = None):
        """Run COMPUTE for explicit inputs (no mutation); returns per-input dicts.
        trace: also return each input's ExecHooks event stream ("events": tuples
        ("mem", kernel, iid, ctaid, tid, space, addr, width, is_store) /
        ("cf", kernel, ctaid, tid, src_block, dst_block), executor.py:108-135),
        recorded on the device by the generic interpreter (sfg_execute_trace)."""
        from .interop import as_testcase
        tcs = [as_testcase(t) for t in tcs]
        n = len(tcs)
        S = self._aux_slot(n)
        self.drain()
        vals_all = np.zeros(n * self.n_args, VAL)
        chld = np.zeros(n, CHILD)
        work = bytearray()
        ro_base = np.zeros(n, np.uint64)
        wbase = np.zeros(n, np.uint64)
        ro_total = 0
        for i, tc in enumerate(tcs):
            vals, _ = pack_values(tc, self.specs)
            wbase[i] = len(work)
            off = 0
            region = bytearray()
            for a, v in enumerate(tc.args):
                if vals[a]["kind"] != 2:
                    continue
                size = max(v.size_override if v.size_override is not None else len(v.data), 0)
                chunk = v.data[:size] + bytes(max(0, size - len(v.data)))
                vals[a]["data_off"] = off
                region += chunk + bytes((-len(chunk)) % 16)
                off += _align16(size)
            region += bytes(int(self.low.prog["named_work_bytes"]) + ov_bytes(int(self.low.prog["ov_cap"])))
            mask = int(self.low.prog["copy_src_mask"])
            for a, v in enumerate(tc.args):     # pristine copies of copy_in sources (sfg_pristine_off)
                if mask >> a & 1:
                    region += v.data + bytes((-len(v.data)) % 16)
            work += region
            chld[i]["it"], chld[i]["parent"], chld[i]["work_bytes"] = iteration0 + i, -1, len(region)
            ro = int(self.low.prog["readout_bytes_fixed"])
            for k in range(int(self.low.prog["n_copyout_arg"])):
                ro += _align16(int(vals[int(self.low.prog["copyout_arg"][k])]["nbytes"]))
            ro_base[i] = ro_total
            ro_total += ro
            chld[i]["readout_bytes"] = ro
            vals_all[i * self.n_args:(i + 1) * self.n_args] = vals
        S.ensure_work(len(work) + 16, self.dev)
        if work:
            S.work[:len(work)].copy_(torch.frombuffer(work, dtype=torch.uint8))
        S.children[:chld.nbytes].copy_(torch.frombuffer(bytearray(chld.tobytes()), dtype=torch.uint8))
        S.vals[:vals_all.nbytes].copy_(torch.frombuffer(bytearray(vals_all.tobytes()), dtype=torch.uint8))
        S.work_base[:n].copy_(torch.from_numpy(wbase.view(np.int64)))
        S.ro_base[:n].copy_(torch.from_numpy(ro_base.view(np.int64)))
        S.readouts = self._u8(ro_total + 16) if self.diff else None
        S.n = n
        torch.cuda.synchronize(self.dev)
        events = None
        if trace:
            tbuf = torch.empty(max(n * trace_cap * 4, 1), dtype=torch.int64, device=self.dev)
            tcnt = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
            self.launches += 1
            _native.check(self.L.sfg_execute_trace(
                self.h, n, S.children.data_ptr(), S.vals.data_ptr(), S.work_base.data_ptr(), S.work.data_ptr(),
                S.verdicts.data_ptr(), S.ecnt.data_ptr(), _ptr(S.readouts), S.ro_base.data_ptr(),
                tbuf.data_ptr(), trace_cap, tcnt.data_ptr(), S.stream.cuda_stream), "execute_trace")
            self.drain()
            cnt = tcnt.cpu().numpy()
            if int(cnt.max(initial=0)) > trace_cap:
                raise DeviceFatal(f"trace buffer overflow ({int(cnt.max())} events > trace_cap {trace_cap})")
            words = tbuf.cpu().numpy().view(np.uint64).reshape(max(n, 1), trace_cap, 4) if n else None
            events = [self._decode_events(words[i, :int(cnt[i])]) for i in range(n)]
        else:
            self._execute(S, n)
        self.drain()
        verd = _np(S.verdicts[:n * VERDICT.itemsize], VERDICT)
        if n and (verd["status"] == ST_OVERLAY).any():   # overlay too small: grow, run again
            self._grow_overlay()
            return self.execute_testcases(tcs, iteration0, trace, trace_cap, id_base)
        E1 = max(self.E, 1)
        ecnt = S.ecnt[:n * E1].cpu().numpy().view(np.uint32).reshape(n, E1)
        rod = S.readouts.cpu().numpy().tobytes() if S.readouts is not None else b""
        out = []
        for i in range(n):
            v = verd[i]
            st = int(v["status"])
            rep = decode_verdict(v, self.low, iteration0 + i, self.base.next_id if id_base is None else id_base) \
                if st == ST_FINDING else None
            readouts = {}
            if S.readouts is not None and st == 0:
                cur = int(ro_base[i])
                for op in self.manifest.phases["compute"]:
                    if op.kind != "copy_out":
                        continue
                    if op.arg_ref >= 0:
                        arg = tcs[i].args[op.arg_ref]
                        if not hasattr(arg, "data"):
                            continue
                        ln = len(arg.data)
                        readouts[f"arg{op.arg_ref}"] = rod[cur:cur + ln]
                    else:
                        ln = op.size
                        readouts[op.name] = rod[cur:cur + ln]
                    cur += _align16(ln)
            out.append({"status": STATUS.get(st, f"fatal{st}"), "report": rep, "retired": int(v["retired"]),
                        "allocs": int(v["allocs"]), "edges": self._edges_row(ecnt[i]), "readouts": readouts,
                        "entered": int(v["entered"])})
            if events is not None:
                out[-1]["events"] = events[i]
        return out

    def _aux_slot(self, n: int) -> Slot:
        """A slot outside the pipelined rounds' ring (explicit executions, tracing)."""
        if getattr(self, "_aux", None) is None or self._aux.cap < n:
            self._aux = Slot(self, max(n, 1024))
        return self._aux

    def _decode_events(self, w: np.ndarray):
        """Device trace words -> ExecHooks argument tuples (csrc/execute.cu layout)."""
        out = []
        spaces = [s.value for s in SPACE_ORDER]
        for w0, w1, w2, w3 in w.tolist():
            kind, kernel, x = w0 & 3, self.low.kernel_names[(w0 >> 16) & 0xFFFF], w0 >> 32
            ctaid, tid = w1 & 0xFFFFFFFF, w1 >> 32
            if kind == 1:
                name, (src, dst) = self.low.edge_names[x]
                out.append(("cf", kernel, ctaid, tid, src, dst))
            else:
                addr = (w3 << 64) | w2
                if addr >= 1 << 127:
                    addr -= 1 << 128
                out.append(("mem", kernel, x, ctaid, tid, spaces[(w0 >> 8) & 0xFF], addr, (w0 >> 3) & 0x1F,
                            bool(w0 & 4)))
        return out

    def close(self):
        """Release the program and every device buffer now (not at garbage
        collection): a following campaign then reuses the memory instead of
        allocating -- cudaMalloc mid-run costs tenths of a second."""
        rl = getattr(self, "round_log", None)
        if getattr(self, "h", None):
            try:
                self.drain()
            except Exception:
                pass
            if rl is not None:
                rl.append(("close_drained", -1, time.perf_counter()))
            self.L.sfg_program_destroy(self.h)
            self.h = None
            if rl is not None:
                rl.append(("close_destroyed", -1, time.perf_counter()))
        self.slots = []
        self._aux = None
        if rl is not None:
            rl.append(("close_slots", -1, time.perf_counter()))
        for name in ("blob", "c_meta", "c_vals", "c_child", "c_data", "edge_total", "ghit", "entered", "counts_run",
                     "ctx_map", "edge_ctx", "ctx_new", "seq_scratch"):
            if hasattr(self, name):
                setattr(self, name, None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
