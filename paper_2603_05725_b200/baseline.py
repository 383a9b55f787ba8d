"""Post-INIT device state: the baseline every fuzz input starts from.

Host-side, once per campaign.  Runs the harness INIT script (allocs, bulk
copies, frees) against a compact allocation registry that follows the
reference allocator (``simt_forge/device_memory.py:397-487``: slot = redzone |
granule-aligned payload | redzone, per-space bump cursor, exact-size free
lists reused lowest-offset first, FIFO quarantine with a byte budget) and
records the result as

* allocation records (all of them, evicted ones too: provenance tags keep
  pointing at them, ``sanitizer.py:174-181``),
* bump cursors, free lists, quarantine order and bytes,
* one payload blob holding every INIT buffer's bytes (uploaded to HBM once;
  inputs read it through the device overlay and never copy it).

This replaces the per-iteration ``image.restore(snapshot)`` of the reference
loop (``campaign.py:729-736``): on the device every input starts from these
immutable tables.

INIT launches run on the device (``init_launch``, supplied by the engine): the
launch's array arguments are materialized here first, exactly as
``PhaseRunner._bind_launch``/``_materialize`` would (campaign.py:440-479: in
binding order, fresh ids, the seed's bytes), so that every byte the launch can
touch is an allocation record of the state so far; the engine runs the launch
on a one-input device program over that state and returns the final bytes of
every live record, which become the records' data.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .manifest import INIT
from .sir import SPACE_ORDER, MemSpace
from .testcase import ArrayValue, FloatValue, IntValue

SPACE_BASE = {MemSpace.GLOBAL: 0x1000_0000, MemSpace.SHARED: 0x2000_0000, MemSpace.LOCAL: 0x3000_0000}


class OutOfSpaceError(Exception):
    pass


class LoweringError(Exception):
    """Harness feature the device path does not lower (raised before any device work)."""


class InitFailure(Exception):
    """INIT produced a finding / error on the seed input (reference: CampaignFatalError)."""


@dataclass(frozen=True)
class MemConfig:
    """Mirror of the reference ``MemConfig`` (device_memory.py:77-121)."""
    global_size: int = 16 * 1024 * 1024
    shared_size: int = 48 * 1024
    local_size: int = 16 * 1024
    shared_scopes: int = 1
    local_scopes: int = 1
    granule: int = 4
    redzone: int = 32
    quarantine_global: int = 1024 * 1024
    quarantine_shared: int = 0
    quarantine_local: int = 0

    def __post_init__(self):
        if self.granule < 1:
            raise ValueError("granule must be >= 1")
        if self.redzone <= 0 or self.redzone % self.granule:
            raise ValueError("redzone must be a positive multiple of the granule")
        for size in (self.global_size, self.shared_size, self.local_size):
            if size <= 0 or size % self.granule:
                raise ValueError("space sizes must be positive multiples of the granule")

    def scope_size(self, sp):
        return {MemSpace.GLOBAL: self.global_size, MemSpace.SHARED: self.shared_size,
                MemSpace.LOCAL: self.local_size}[sp]

    def scopes(self, sp):
        return {MemSpace.GLOBAL: 1, MemSpace.SHARED: self.shared_scopes, MemSpace.LOCAL: self.local_scopes}[sp]

    def qcap(self, sp):
        return {MemSpace.GLOBAL: self.quarantine_global, MemSpace.SHARED: self.quarantine_shared,
                MemSpace.LOCAL: self.quarantine_local}[sp]


@dataclass
class Record:
    alloc_id: int
    space: MemSpace
    base: int
    size: int
    slot_start: int
    slot_end: int
    label: str
    freed: bool = False
    resident: bool = True
    data: bytearray = field(default_factory=bytearray)


@dataclass
class Baseline:
    records: list
    named: dict                 # name -> (addr, id, record index)
    cursor: dict
    qbytes: dict
    quarantine: list            # record indices, FIFO
    free_entries: list          # (offset within space, slot size, space)
    next_id: int
    blob: bytes
    phys: list                  # blob offset per record


def _up(n: int, a: int) -> int:
    return (n + a - 1) // a * a


INTERNAL_ARG = "\0arg{}"    # named handle of an array argument materialized by an INIT launch


def build_baseline(manifest, seed_tc, mem: MemConfig, init_launch=None) -> Baseline:
    """``init_launch(op, state, names) -> {name: bytes}`` runs one INIT launch on the
    device over ``state`` (a Baseline of everything so far) and returns the final
    payload of each named live record in ``names``; it raises InitFailure when the
    launch stops on a finding or the budget."""
    recs: list[Record] = []
    cursor = {sp: 0 for sp in SPACE_ORDER}
    qbytes = {sp: 0 for sp in SPACE_ORDER}
    quar: list[int] = []
    free: list = []
    named: dict = {}
    next_id = 1

    materialized: dict = {}        # arg index -> record index (INIT launches)

    def live_at(addr: int, n: int):
        for j, r in enumerate(recs):
            if r.resident and not r.freed and r.base <= addr and addr + n <= r.base + r.size:
                return j
        return None

    def alloc(sp, size: int, label: str) -> int:
        """_alloc_common (device_memory.py:407-440), scope 0; size 0 = alloc_empty."""
        nonlocal next_id
        slot = mem.redzone + _up(size, mem.granule) + mem.redzone
        cands = [k for k, e in enumerate(free) if e[1] == slot and e[2] == sp]
        if cands:
            k = min(cands, key=lambda j: free[j][0])
            off = free.pop(k)[0]
        else:
            if cursor[sp] + slot > mem.scope_size(sp):
                raise OutOfSpaceError(f"{sp.value} scope 0: need {slot} bytes, "
                                      f"{mem.scope_size(sp) - cursor[sp]} remain")
            off = cursor[sp]
            cursor[sp] += slot
        start = SPACE_BASE[sp] + off
        recs.append(Record(next_id, sp, start + mem.redzone, size, start, start + slot, label,
                           data=bytearray(size)))
        next_id += 1
        return len(recs) - 1

    def state() -> Baseline:
        blob, phys = bytearray(), []
        for r in recs:
            phys.append(len(blob))
            blob += r.data + bytes((-len(r.data)) % 16)
        return Baseline(list(recs), dict(named), dict(cursor), dict(qbytes), list(quar), list(free), next_id,
                        bytes(blob) or b"\0", phys)

    for op in manifest.phases[INIT]:
        if op.kind == "sync":
            continue
        if op.kind == "alloc":
            if op.size <= 0:
                raise InitFailure(f"allocation size must be positive, got {op.size}")
            j = alloc(op.space, op.size, op.name)
            named[op.name] = (recs[j].base, recs[j].alloc_id, j)
        elif op.kind == "copy_in":
            addr = named[op.name][0]
            form, payload = op.source
            if form == "zeros":
                data = bytes(int(payload, 0))
            elif form == "seq32":
                data = np.arange(int(payload, 0), dtype="<u4").tobytes()
            elif form == "hex":
                data = bytes.fromhex(payload)
            else:
                v = seed_tc.args[int(payload)]
                data = (v.data if isinstance(v, ArrayValue) else
                        (v.value & 0xFFFFFFFF).to_bytes(4, "little") if isinstance(v, IntValue) else
                        v.bits.to_bytes(4, "little"))
            if not data:
                continue
            j = live_at(addr, len(data))
            if j is None:
                raise InitFailure("init phase failed on the seed input: finding")
            r = recs[j]
            r.data[addr - r.base:addr - r.base + len(data)] = data
        elif op.kind == "copy_out":
            if op.arg_ref >= 0:       # only after an INIT launch materialized it (campaign.py:517-520)
                if op.arg_ref in materialized:
                    r = recs[materialized[op.arg_ref]]
                    n = len(seed_tc.args[op.arg_ref].data)
                    if n and live_at(r.base, n) is None:
                        raise InitFailure("init phase failed on the seed input: finding")
                continue
            addr = named[op.name][0]
            if op.size and live_at(addr, op.size) is None:
                raise InitFailure("init phase failed on the seed input: finding")
        elif op.kind == "free":
            addr = named[op.name][0]
            hits = [j for j, r in enumerate(recs) if r.resident and r.base == addr]
            if not hits or recs[hits[0]].freed:
                raise InitFailure("init phase failed on the seed input: finding")
            r = recs[hits[0]]
            r.freed = True
            quar.append(hits[0])
            qbytes[r.space] += r.slot_end - r.slot_start
            while qbytes[r.space] > mem.qcap(r.space):
                qi = next(q for q, j in enumerate(quar) if recs[j].space == r.space)
                v = recs[quar.pop(qi)]
                v.resident = False
                free.append((v.slot_start - SPACE_BASE[v.space], v.slot_end - v.slot_start, v.space))
                qbytes[v.space] -= v.slot_end - v.slot_start
        elif op.kind == "launch":
            if init_launch is None:
                raise LoweringError("INIT-phase launches need the device (init_launch)")
            binds = []
            for b in op.bindings:
                v = seed_tc.args[b[1]] if b[0] == "arg" else None
                if isinstance(v, ArrayValue):      # _bind_launch / _materialize, binding order
                    k = b[1]
                    if v.base_offset:
                        raise LoweringError("INIT launch of an array with a base offset")
                    if k not in materialized:
                        size = v.size_override if v.size_override is not None else len(v.data)
                        j = alloc(v.space, max(size, 0), f"arg{k}")
                        if size > 0:
                            recs[j].data[:] = v.data[:size]
                        materialized[k] = j
                        named[INTERNAL_ARG.format(k)] = (recs[j].base, recs[j].alloc_id, j)
                    binds.append(("buf", INTERNAL_ARG.format(k)))
                else:
                    binds.append(b)
            live = [n for n, (_, _, j) in named.items() if recs[j].resident and not recs[j].freed]
            out = init_launch(replace(op, bindings=tuple(binds)), state(), live)
            for n, data in out.items():
                r = recs[named[n][2]]
                r.data[:] = data
    blob = bytearray()
    phys = []
    for r in recs:
        phys.append(len(blob))
        blob += r.data + bytes((-len(r.data)) % 16)
    return Baseline(recs, named, cursor, qbytes, quar, free, next_id, bytes(blob) or b"\0", phys)


def term_frees_clean(b: Baseline, term_ops) -> bool:
    """A TERM script of frees (and syncs) only, on the post-INIT state, frees live
    allocations or skips already-freed ones (campaign.py:538-541) -- no report.
    Anything else is run on the device (engine.DeviceCampaign.run_term)."""
    seen = set()
    for op in term_ops:
        if op.kind == "sync":
            continue
        if op.kind != "free" or op.name not in b.named or op.name in seen:
            return False     # (a repeated free may meet an evicted record: the device decides)
        seen.add(op.name)
        addr = b.named[op.name][0]
        if not any(r.resident and r.base == addr for r in b.records):
            return False
    return True


def record_table(b: Baseline, labels: list):
    from .lowering import MAX_BASE_RECS, MAX_FREE, REC, LoweringError
    from .sir import SPACE_INDEX
    if len(b.records) > MAX_BASE_RECS or len(b.free_entries) > MAX_FREE:
        raise LoweringError("INIT leaves more allocation records / free slots than the device tables hold")
    arr = np.zeros(max(len(b.records), 1), REC)
    for j, r in enumerate(b.records):
        arr[j]["base"], arr[j]["size"] = r.base, r.size
        arr[j]["slot_start"], arr[j]["slot_end"] = r.slot_start, r.slot_end
        arr[j]["phys"], arr[j]["id"] = b.phys[j], r.alloc_id
        arr[j]["label"] = labels.index(r.label)
        arr[j]["space"], arr[j]["state"] = SPACE_INDEX[r.space], int(r.freed)
        arr[j]["resident"] = int(r.resident)
    return arr
