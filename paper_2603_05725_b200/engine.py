"""Device round driver: one batched round of the fuzzing inner loop on a GPU.

A *round* is R consecutive fuzz inputs ``it0 .. it0+R-1`` of the batched-round
contract: every input schedules a parent from the corpus as it
stood at the round start, mutates with its own Philox stream, executes its
COMPUTE phase on the post-INIT baseline, and is absorbed in ``it`` order.
All of it runs as stream-ordered kernels from ``libsfg_b200.so``; torch only
holds device memory and provides the stream.  Host work per round: three
small device->host reads (work-arena size, stop/fatal/admission scalars,
dedupe-key table) and building reference-typed objects for the (rare) new
findings and admitted children.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .baseline import MemConfig, OutOfSpaceError, build_baseline, record_table
from .coverage import CoverageMap
from .findings import FindingsLog
from .lowering import (CHILD, ENTRY, KEYBASE, ST_COUNTER, ST_FINDING, ST_LANE_RECS, ST_OUT_OF_SPACE, ST_OVERLAY,
                       ST_ZERO_ALLOC, VAL, VERDICT, Lowered, LoweringError, decode_op, decode_verdict,
                       pack_values, unpack_values)
from .testcase import MutationError, TestCase

U32_NONE = 0xFFFFFFFF


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


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _np(t: torch.Tensor, dtype) -> np.ndarray:
    return t.detach().cpu().numpy().view(dtype)


class RoundResult:
    """Device buffers + host scalars of one executed round."""

    def __init__(self, it0, n, stop, executed, admitted, new_keys):
        self.it0, self.n, self.stop, self.executed = it0, n, stop, executed
        self.n_admitted = admitted
        self.new_keys = new_keys


class DeviceCampaign:
    def __init__(self, manifest, *, master_seed=1, mem: MemConfig | None = None,
                 mutation: MutationConfig | None = None, budget=1_000_000, window=256, recent_weight=4.0,
                 diff_readback=False, stop_on_first_finding=False, stop_bug_class=None, device=None,
                 extra_seeds=(), ids_reset_per_input=False):
        if not torch.cuda.is_available():
            raise _native.NativeError("no CUDA device: the fuzzing inner loop runs only on the GPU")
        self.L = _native.lib()
        self.dev = torch.device(device or "cuda")
        self.manifest = manifest
        self.mem = mem or MemConfig()
        self.mutation = mutation or MutationConfig()
        self.master_seed = master_seed
        self.seed_tc = manifest.seed(master_seed)
        self.base = build_baseline(manifest, self.seed_tc, self.mem)
        stop_class = None
        if stop_bug_class is not None:
            stop_class = getattr(stop_bug_class, "value", str(stop_bug_class))
        self.low = Lowered(manifest, self.base, mem=self.mem, mutation=self.mutation, master_seed=master_seed,
                           budget=budget, window=window, recent_weight=recent_weight,
                           diff_readback=diff_readback, stop_first=stop_on_first_finding, stop_class=stop_class)
        self.specs = manifest.argspecs
        self.n_args = len(self.specs)
        self.C = len(self.low.int_args)
        if self.C > 8:
            raise LoweringError("more than 8 i32 arguments")
        self.E = self.low.n_edges
        self.K = self.low.n_keys
        recs = record_table(self.base, self.low.labels)
        self.blob = torch.frombuffer(bytearray(self.base.blob), dtype=torch.uint8).to(self.dev)
        h = ctypes.c_void_p()
        P = self.low.prog_bytes()
        _native.check(self.L.sfg_program_create(
            P, len(P), self.low.ins.ctypes.data, len(self.low.ins), self.low.hostops.ctypes.data,
            len(self.low.hostops), self.low.binds.ctypes.data, len(self.low.binds), recs.ctypes.data, len(recs),
            self.low.const_blob, len(self.low.const_blob), self.blob.data_ptr(), ctypes.byref(h)),
            "sfg_program_create")
        self.h = h
        # global campaign state on device
        self.edge_total = torch.zeros(max(self.E, 1), dtype=torch.int64, device=self.dev)
        self.ghit = torch.zeros(max(self.E, 1), dtype=torch.uint8, device=self.dev)
        self.entered = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.counts_base = torch.zeros(max(self.C, 1), dtype=torch.int64, device=self.dev)
        self.next_alloc_id = self.base.next_id
        self.ids_reset = ids_reset_per_input   # reinit mode: every input gets a fresh image
        self.findings = FindingsLog()
        self.key_strings: dict[int, str] = {}
        # corpus (device) + host mirror
        self.cap = 0
        self.data_cap = 0
        self.n_corpus = 0
        self.corpus_bytes = 0
        self.host_entries: list = []     # (TestCase, admitted_iteration, is_seed)
        seeds = [self.seed_tc] + list(extra_seeds)
        self._grow_corpus(max(64, len(seeds) * 2), 1 << 16)
        self._upload_seeds(seeds)
        self.n_seeds = len(seeds)
        self._round_cap = 0
        self._work_cap = 0
        self.rounds = 0
        self.launches = 0          # kernels launched through the C ABI (bench evidence)
        self.timing = False        # record CUDA events around the execute kernel
        self.last_exec_events = None

    # ---- buffers ---------------------------------------------------------------------
    def _u8(self, n):
        return torch.empty(max(int(n), 16), dtype=torch.uint8, device=self.dev)

    def _grow_corpus(self, cap, data_cap):
        cap, data_cap = max(cap, self.cap), max(data_cap, self.data_cap)
        if cap == self.cap and data_cap == self.data_cap:
            return
        meta = self._u8(cap * ENTRY.itemsize)
        vals = self._u8(cap * self.n_args * VAL.itemsize)
        chld = self._u8(cap * CHILD.itemsize)
        data = self._u8(data_cap)
        if self.cap:
            meta[:self.cap * ENTRY.itemsize].copy_(self.c_meta[:self.cap * ENTRY.itemsize])
            vals[:self.cap * self.n_args * VAL.itemsize].copy_(self.c_vals[:self.cap * self.n_args * VAL.itemsize])
            chld[:self.cap * CHILD.itemsize].copy_(self.c_child[:self.cap * CHILD.itemsize])
            data[:self.data_cap].copy_(self.c_data[:self.data_cap])
        self.c_meta, self.c_vals, self.c_child, self.c_data = meta, vals, chld, data
        self.cap, self.data_cap = cap, data_cap

    def _upload_seeds(self, seeds):
        metas = np.zeros(len(seeds), ENTRY)
        allv = []
        blob = bytearray()
        for j, tc in enumerate(seeds):
            vals, payload = pack_values(tc, self.specs)
            vals["data_off"] += np.where(vals["kind"] == 2, len(blob), 0).astype(np.uint64)
            blob += payload
            allv.append(vals)
            metas[j] = (0, tc.rng_seed & ((1 << 64) - 1), 1, -1, 0)
            self.host_entries.append((tc, 0, True))
        self._grow_corpus(len(seeds) * 2, len(blob) * 2 + 4096)
        v = np.concatenate(allv)
        self.c_meta[:metas.nbytes].copy_(torch.frombuffer(bytearray(metas.tobytes()), dtype=torch.uint8))
        self.c_vals[:v.nbytes].copy_(torch.frombuffer(bytearray(v.tobytes()), dtype=torch.uint8))
        if blob:
            self.c_data[:len(blob)].copy_(torch.frombuffer(blob, dtype=torch.uint8))
        self.n_corpus = len(seeds)
        self.corpus_bytes = len(blob)

    def _ensure_round(self, n):
        if n <= self._round_cap:
            return
        n = max(n, 1024)
        C, E = max(self.C, 1), max(self.E, 1)
        i64 = lambda m: torch.empty(max(m, 1), dtype=torch.int64, device=self.dev)  # noqa: E731
        i32 = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=self.dev)  # noqa: E731
        self.r_parent = i32(n)
        self.r_picks = self._u8(n * 3)
        self.r_flags = i32(n * C)
        self.r_prefix = i64(n * C)
        self.r_children = self._u8(n * CHILD.itemsize)
        self.r_vals = self._u8(n * self.n_args * VAL.itemsize)
        self.r_work_base = i64(n)
        self.r_ro_base = i64(n)
        self.r_verdicts = self._u8(n * VERDICT.itemsize)
        self.r_ecnt = i32(n * E)
        self.r_overlay = i64(n * 32) if self.low.overlay else None
        self.r_allocs = i64(n)
        self.r_allocs_prefix = i64(n)
        self.r_admit = i64(n)
        self.r_pos = i64(n)
        self.r_bytes = i64(n)
        self.r_boff = i64(n)
        self.r_sel = i32(n)
        self.r_dst_off = i64(n * self.n_args)
        self.r_tmp = i64((n + 2047) // 2048 + 8)
        self.r_tot = i64(16)
        self.r_scalars = i32(2)
        self.r_first = i32(E)
        self.r_kfirst = i32(self.K)
        self.r_kcount = i64(self.K)
        self._round_cap = n

    def _ensure_work(self, nbytes):
        if nbytes > self._work_cap:
            self._work_cap = int(nbytes * 1.25) + 4096
            self.r_work = self._u8(self._work_cap)

    def corpus_dev(self) -> CorpusDev:
        return CorpusDev(self.c_meta.data_ptr(), self.c_vals.data_ptr(), self.c_data.data_ptr(),
                         self.n_corpus, self.n_seeds)

    def _scan64(self, src, n, stride, col, out, out_stride, total_slot):
        self.launches += 3
        _native.check(self.L.sfg_scan_u64(src.data_ptr(), n, stride, col, out.data_ptr(), out_stride, 0,
                                          self.r_tmp.data_ptr(), self.r_tot.data_ptr() + 8 * total_slot,
                                          _stream()), "scan")

    def new_worker(self):
        """Reference workers (campaign.py:712-730) get a fresh MutationSchedule and a fresh
        image: rotation counts and alloc ids restart; corpus/findings/coverage are shared."""
        self.counts_base.zero_()
        self.next_alloc_id = self.base.next_id

    def _id_base(self, prefix: int) -> int:
        return self.base.next_id if self.ids_reset else self._round_id0 + prefix

    # ---- one round ---------------------------------------------------------------------
    def run_round(self, it0: int, n: int) -> RoundResult:
        L, hp, s = self.L, self.h, _stream()
        self._ensure_round(n)
        cd = self.corpus_dev()
        if it0 + n - 1 >= 2 and self.low.prog["n_mutable"] == 0:
            raise MutationError("no mutable arguments")
        C = self.C
        self.launches += 3 + 3 * C
        _native.check(L.sfg_plan(hp, ctypes.byref(cd), it0, n, self.r_parent.data_ptr(), self.r_picks.data_ptr(),
                                 self.r_flags.data_ptr(), s), "plan")
        for c in range(C):
            _native.check(L.sfg_scan_u32(self.r_flags.data_ptr(), n, C, c, self.r_prefix.data_ptr(), C, c,
                                         self.r_tmp.data_ptr(), self.r_tot.data_ptr() + 8 * (8 + c % 8), s),
                          "scan flags")
        _native.check(L.sfg_mutate(hp, ctypes.byref(cd), it0, n, self.r_prefix.data_ptr(),
                                   self.counts_base.data_ptr(), self.r_children.data_ptr(), self.r_vals.data_ptr(),
                                   s), "mutate")
        cw = CHILD.itemsize // 8
        self._scan64(self.r_children.view(torch.int64), n, cw, CHILD.fields["work_bytes"][1] // 8,
                     self.r_work_base, 1, 0)
        if self.low.prog["diff_readback"]:
            self._scan64(self.r_children.view(torch.int64), n, cw, CHILD.fields["readout_bytes"][1] // 8,
                         self.r_ro_base, 1, 1)
        tot = self.r_tot[:2].cpu()
        self._ensure_work(int(tot[0]))
        ro = self._u8(int(tot[1])) if self.low.prog["diff_readback"] else None
        self.r_readouts = ro
        _native.check(L.sfg_apply(hp, ctypes.byref(cd), n, self.r_children.data_ptr(), self.r_vals.data_ptr(),
                                  self.r_work_base.data_ptr(), self.r_work.data_ptr(), s), "apply")
        self._execute(n)
        return self._triage(it0, n)

    def _execute(self, n):
        self.launches += 1
        if self.timing:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        _native.check(self.L.sfg_execute(
            self.h, n, self.r_children.data_ptr(), self.r_vals.data_ptr(), self.r_work_base.data_ptr(),
            self.r_work.data_ptr(), self.r_verdicts.data_ptr(), self.r_ecnt.data_ptr(), _ptr(self.r_readouts),
            self.r_ro_base.data_ptr(), _ptr(self.r_overlay), _stream()), "execute")
        if self.timing:
            ev[1].record()
            self.last_exec_events = ev

    def _triage(self, it0, n) -> RoundResult:
        L, hp, s = self.L, self.h, _stream()
        self.launches += 4
        self.r_scalars.fill_(-1)
        self.r_first.fill_(-1)
        self.r_kfirst.fill_(-1)
        self.r_kcount.zero_()
        _native.check(L.sfg_triage(hp, n, self.r_verdicts.data_ptr(), self.r_ecnt.data_ptr(),
                                   self.r_children.data_ptr(), self.r_scalars.data_ptr(), self.r_first.data_ptr(),
                                   self.edge_total.data_ptr(), self.r_kfirst.data_ptr(), self.r_kcount.data_ptr(),
                                   self.entered.data_ptr(), self.r_allocs.data_ptr(), self.ghit.data_ptr(),
                                   self.r_admit.data_ptr(), s), "triage")
        self._scan64(self.r_admit, n, 1, 0, self.r_pos, 1, 2)
        self._scan64(self.r_allocs, n, 1, 0, self.r_allocs_prefix, 1, 3)
        sc = self.r_scalars.cpu().numpy().view(np.uint32)
        tot = self.r_tot[:16].cpu().numpy().view(np.uint64)
        stop, fatal = int(sc[0]), int(sc[1])
        if fatal != U32_NONE and fatal <= stop:
            self._raise_fatal(fatal)
        executed = n if stop == U32_NONE else stop + 1
        n_adm = int(tot[2])
        self._round_id0 = self.next_alloc_id
        if n_adm:
            self._admit(n, n_adm)
        _native.check(L.sfg_commit(hp, self.edge_total.data_ptr(), self.ghit.data_ptr(), s), "commit")
        new_keys = self._absorb_findings(it0)
        self.next_alloc_id += int(tot[3])
        if stop == U32_NONE and self.C:
            self.counts_base[:self.C] += self.r_tot[8:8 + self.C]
        self.rounds += 1
        return RoundResult(it0, n, None if stop == U32_NONE else stop, executed, n_adm, new_keys)

    def _raise_fatal(self, i):
        v = _np(self.r_verdicts[i * VERDICT.itemsize:(i + 1) * VERDICT.itemsize], VERDICT)[0]
        st = int(v["status"])
        if st == ST_OUT_OF_SPACE:
            raise OutOfSpaceError(f"input {i}: allocation does not fit its space")
        if st == ST_ZERO_ALLOC:
            raise ValueError("allocation size must be positive")
        raise DeviceFatal({ST_LANE_RECS: "per-input allocation table overflow",
                           ST_OVERLAY: "per-input INIT-buffer write overlay overflow",
                           ST_COUNTER: "per-input edge counter overflow"}.get(st, f"status {st}"))

    def _admit(self, n, n_adm):
        L, hp, s = self.L, self.h, _stream()
        self.launches += 3
        _native.check(L.sfg_child_bytes(hp, self.r_vals.data_ptr(), self.r_admit.data_ptr(), n,
                                        self.r_bytes.data_ptr(), s), "child_bytes")
        self._scan64(self.r_bytes, n, 1, 0, self.r_boff, 1, 4)
        nbytes = int(self.r_tot[4].item())
        self._grow_corpus(max(self.cap, (self.n_corpus + n_adm) * 2),
                          max(self.data_cap, (self.corpus_bytes + nbytes) * 2))
        cd = self.corpus_dev()
        _native.check(L.sfg_compact(hp, self.r_children.data_ptr(), self.r_vals.data_ptr(), self.r_admit.data_ptr(),
                                    self.r_pos.data_ptr(), self.r_boff.data_ptr(), n, self.n_corpus,
                                    self.corpus_bytes, self.c_meta.data_ptr(), self.c_vals.data_ptr(),
                                    self.c_child.data_ptr(), self.r_sel.data_ptr(), self.r_dst_off.data_ptr(), s),
                      "compact")
        _native.check(L.sfg_regen(hp, ctypes.byref(cd), n_adm, self.r_sel.data_ptr(), self.r_children.data_ptr(),
                                  self.r_vals.data_ptr(), self.r_dst_off.data_ptr(), self.c_data.data_ptr(), s),
                      "regen")
        first = self.n_corpus
        self.n_corpus += n_adm
        self.corpus_bytes += nbytes
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
        for j in range(hi - lo):
            args = unpack_values(vals[j * self.n_args:(j + 1) * self.n_args], data, base)
            parent_tc = self.host_entries[int(meta[j]["parent"])][0]
            ops = tuple(decode_op(chld[j]["ops"][k]) for k in range(int(chld[j]["n_ops"])))
            tc = TestCase(args, int(meta[j]["rng_seed"]), parent_tc.id, ops)
            self.host_entries.append((tc, int(meta[j]["admitted_iteration"]), False))

    def _absorb_findings(self, it0):
        kc = self.r_kcount.cpu().numpy()
        hot = np.nonzero(kc)[0]
        if not len(hot):
            return []
        kf = self.r_kfirst.cpu().numpy().view(np.uint32)
        fresh = []
        for k in hot:
            ks = self.key_strings.get(int(k))
            if ks is not None and ks in self.findings:
                self.findings.bump(ks, int(kc[k]))
            else:
                fresh.append((int(kf[k]), int(k)))
        fresh.sort()
        out = []
        if fresh:
            idx = [i for i, _ in fresh]
            vt = _np(self.r_verdicts.view(-1, VERDICT.itemsize)[idx].reshape(-1), VERDICT)
            ap = self.r_allocs_prefix[idx].cpu().numpy()
            for j, (i, k) in enumerate(fresh):
                rep = decode_verdict(vt[j], self.low, it0 + i, self._id_base(int(ap[j])))
                self.key_strings[k] = rep.dedupe_key
                self.findings.add_many(rep, int(kc[k]))
                out.append((i, rep))
        return out

    # ---- bench / e2e helpers ----------------------------------------------------------
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

    def load_corpus_from_host(self, host):
        """Re-upload the corpus from pinned host buffers (stream-ordered H2D copies)."""
        for t, h in zip((self.c_meta, self.c_vals, self.c_child, self.c_data), host):
            t[:h.numel()].copy_(h, non_blocking=True)

    def algorithmic_exec_bytes(self) -> int:
        """Unavoidable off-chip bytes of one exec in the execute kernel: the child's
        argument payload read once (SURVEY.md §8(d) C_write counterpart), its 64-byte
        verdict and a 4*ceil(E/32)-byte edge-hit bitmap written."""
        seed = self.host_entries[0][0]
        payload = sum(len(v.data) if hasattr(v, "data") else 4 for v in seed.args)
        return payload + 64 + 4 * ((self.E + 31) // 32)

    def retired_mean(self, n: int) -> float:
        v = _np(self.r_verdicts[:n * VERDICT.itemsize], VERDICT)
        return float(v["retired"].astype(np.float64).mean())

    # ---- views for tests / reporting ----------------------------------------------------
    def coverage_map(self) -> CoverageMap:
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

    def round_records(self, res: RoundResult):
        """Per-input records of the last round (same shape as oracle.loop records)."""
        n = res.executed
        s = _stream()
        vals = _np(self.r_vals[:n * self.n_args * VAL.itemsize], VAL)
        chld = _np(self.r_children[:n * CHILD.itemsize], CHILD)
        verd = _np(self.r_verdicts[:n * VERDICT.itemsize], VERDICT)
        ecnt = self.r_ecnt[:n * max(self.E, 1)].cpu().numpy().view(np.uint32).reshape(n, max(self.E, 1))
        admit = self.r_admit[:n].cpu().numpy()
        aprefix = self.r_allocs_prefix[:n].cpu().numpy()
        tcs = self.child_testcases(list(range(n)))
        recs = []
        for i in range(n):
            c = chld[i]
            p = int(c["parent"])
            tc = tcs[i]
            v = verd[i]
            st = int(v["status"])
            rep = decode_verdict(v, self.low, int(c["it"]), self._id_base(int(aprefix[i]))) if st == ST_FINDING else None
            edges = {}
            for e in np.nonzero(ecnt[i][:self.E])[0]:
                name, (a, b) = self.low.edge_names[e]
                edges.setdefault(name, []).append([a, b, int(ecnt[i][e])])
            recs.append({"it": int(c["it"]), "parent": p, "child": tc,
                         "status": {0: "ok", 1: "finding", 2: "budget"}.get(st, f"fatal{st}"),
                         "retired": int(v["retired"]), "allocs": int(v["allocs"]),
                         "edges": {k: sorted(x) for k, x in edges.items()},
                         "report": rep.to_line() if rep else None, "admitted": bool(admit[i])})
        return recs

    def child_testcases(self, idx):
        """Reference TestCase objects for round inputs ``idx``: payloads regenerated
        on the device from (parent, ops) with the product kernel, then decoded."""
        n = len(idx)
        if n == 0:
            return []
        s = _stream()
        sel_np = np.asarray(idx, np.int32)
        vals = _np(self.r_vals.view(-1, VAL.itemsize * self.n_args)[torch.from_numpy(sel_np).long().to(self.dev)]
                   .reshape(-1), VAL)
        chld = _np(self.r_children.view(-1, CHILD.itemsize)[torch.from_numpy(sel_np).long().to(self.dev)]
                   .reshape(-1), CHILD)
        offs = np.zeros(n * self.n_args, np.uint64)
        cur = 0
        for j in range(n):
            for a in range(self.n_args):
                v = vals[j * self.n_args + a]
                if v["kind"] == 2:
                    offs[j * self.n_args + a] = cur
                    cur += (int(v["nbytes"]) + 15) // 16 * 16
        dst = self._u8(cur + 16)
        sel = torch.from_numpy(sel_np).to(self.dev)
        doff = torch.from_numpy(offs.view(np.int64)).to(self.dev)
        cd = self.corpus_dev()
        self.launches += 1
        _native.check(self.L.sfg_regen(self.h, ctypes.byref(cd), n, sel.data_ptr(), self.r_children.data_ptr(),
                                       self.r_vals.data_ptr(), doff.data_ptr(), dst.data_ptr(), s), "regen")
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
    def execute_testcases(self, tcs, iteration0: int = 0):
        """Run COMPUTE for explicit inputs (no mutation); returns per-input dicts."""
        n = len(tcs)
        self._ensure_round(n)
        vals_all = np.zeros(n * self.n_args, VAL)
        chld = np.zeros(n, CHILD)
        work = bytearray()
        ro_base = np.zeros(n, np.uint64)
        ro_total = 0
        wbase = np.zeros(n, np.uint64)
        for i, tc in enumerate(tcs):
            vals, _ = pack_values(tc, self.specs)
            wbase[i] = len(work)
            off = 0
            region = bytearray()
            for a, v in enumerate(tc.args):
                if vals[a]["kind"] != 2:
                    continue
                size = v.size_override if v.size_override is not None else len(v.data)
                size = max(size, 0)
                chunk = v.data[:size] + bytes(max(0, size - len(v.data)))
                vals[a]["data_off"] = off
                region += chunk + bytes((-len(chunk)) % 16)
                off += (size + 15) // 16 * 16
            region += bytes(int(self.low.prog["named_work_bytes"]))
            work += region
            chld[i]["it"] = iteration0 + i
            chld[i]["parent"] = -1
            chld[i]["work_bytes"] = len(region)
            ro = int(self.low.prog["readout_bytes_fixed"])
            for k in range(int(self.low.prog["n_copyout_arg"])):
                ro += (int(vals[int(self.low.prog["copyout_arg"][k])]["nbytes"]) + 15) // 16 * 16
            ro_base[i] = ro_total
            ro_total += ro
            chld[i]["readout_bytes"] = ro
            vals_all[i * self.n_args:(i + 1) * self.n_args] = vals
        self._ensure_work(len(work) + 16)
        self.r_work[:len(work)].copy_(torch.frombuffer(work, dtype=torch.uint8)) if work else None
        self.r_children[:chld.nbytes].copy_(torch.frombuffer(bytearray(chld.tobytes()), dtype=torch.uint8))
        self.r_vals[:vals_all.nbytes].copy_(torch.frombuffer(bytearray(vals_all.tobytes()), dtype=torch.uint8))
        self.r_work_base[:n].copy_(torch.from_numpy(wbase.view(np.int64)))
        self.r_ro_base[:n].copy_(torch.from_numpy(ro_base.view(np.int64)))
        self.r_readouts = self._u8(ro_total + 16) if self.low.prog["diff_readback"] else None
        self._execute(n)
        verd = _np(self.r_verdicts[:n * VERDICT.itemsize], VERDICT)
        ecnt = self.r_ecnt[:n * max(self.E, 1)].cpu().numpy().view(np.uint32).reshape(n, max(self.E, 1))
        rod = self.r_readouts.cpu().numpy().tobytes() if self.r_readouts is not None else b""
        out = []
        for i in range(n):
            v = verd[i]
            st = int(v["status"])
            rep = decode_verdict(v, self.low, iteration0 + i, self.base.next_id) if st == ST_FINDING else None
            edges = {}
            for e in np.nonzero(ecnt[i][:self.E])[0]:
                name, (a, b) = self.low.edge_names[e]
                edges.setdefault(name, []).append([a, b, int(ecnt[i][e])])
            readouts = {}
            if self.r_readouts is not None and st == 0:
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
                    cur += (ln + 15) // 16 * 16
            out.append({"status": {0: "ok", 1: "finding", 2: "budget"}.get(st, f"fatal{st}"),
                        "report": rep, "retired": int(v["retired"]), "allocs": int(v["allocs"]),
                        "edges": {k: sorted(x) for k, x in edges.items()}, "readouts": readouts,
                        "entered": int(v["entered"])})
        return out

    def close(self):
        if getattr(self, "h", None):
            self.L.sfg_program_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
