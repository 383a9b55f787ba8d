"""ORACLE (test infrastructure): simulated device memory + sanitizer, restated.

Memory model follows ``simt_forge/device_memory.py``: three flat spaces
(:41-45), slot = redzone | granule-aligned payload | redzone (:407-440), shadow
codes (:33-36, :347-366), FIFO quarantine with byte budget and exact-size free
lists (:442-487), payload/slot resolution (:491-517), sanitized host copies
(:527-547) and snapshot/restore of the post-INIT state (:551-618; here a plain
deep copy plus dirty-chunk tracking for the byte arrays).

The classifier follows ``simt_forge/sanitizer.py``: ``_scan_shadow`` :102-142,
``check_access`` :145-187, ``check_host_access`` :190-196,
``invalid_free_report`` :199-205.
"""

from __future__ import annotations

import copy
from bisect import bisect_right, insort
from dataclasses import dataclass

from paper_2603_05725_b200.findings import HOST, BugClass, BugReport
from paper_2603_05725_b200.sir import SPACE_ORDER, MemSpace

SH_OK, SH_RZ, SH_FREED, SH_UNALLOC = 0x00, 0xFA, 0xFD, 0xFF
SPACE_BASE = {MemSpace.GLOBAL: 0x1000_0000, MemSpace.SHARED: 0x2000_0000,
              MemSpace.LOCAL: 0x3000_0000}
CHUNK = 256


class OutOfSpaceError(Exception):
    pass


class InvalidFreeError(Exception):
    def __init__(self, addr: int, reason: str):
        super().__init__(f"invalid free of 0x{addr:x}: {reason}")
        self.addr = addr
        self.reason = reason


@dataclass(frozen=True)
class MemCfg:
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

    def scope_size(self, sp):
        return {MemSpace.GLOBAL: self.global_size, MemSpace.SHARED: self.shared_size,
                MemSpace.LOCAL: self.local_size}[sp]

    def scopes(self, sp):
        return {MemSpace.GLOBAL: 1, MemSpace.SHARED: self.shared_scopes,
                MemSpace.LOCAL: self.local_scopes}[sp]

    def total(self, sp):
        return self.scope_size(sp) * self.scopes(sp)

    def qcap(self, sp):
        return {MemSpace.GLOBAL: self.quarantine_global, MemSpace.SHARED: self.quarantine_shared,
                MemSpace.LOCAL: self.quarantine_local}[sp]


@dataclass
class Rec:
    alloc_id: int
    space: MemSpace
    scope: int
    base: int
    size: int
    state: str
    label: str
    slot_start: int
    slot_end: int


def _up(n: int, a: int) -> int:
    return (n + a - 1) // a * a


class Image:
    def __init__(self, cfg: MemCfg | None = None):
        self.cfg = cfg or MemCfg()
        c = self.cfg
        self.mem = {sp: bytearray(c.total(sp)) for sp in SPACE_ORDER}
        self.shadow = {sp: bytearray([SH_UNALLOC]) * (c.total(sp) // c.granule) for sp in SPACE_ORDER}
        self.cursor = {(sp, s): s * c.scope_size(sp) for sp in SPACE_ORDER for s in range(c.scopes(sp))}
        self.records: dict[int, Rec] = {}
        self.rows = {sp: [] for sp in SPACE_ORDER}       # sorted (base, id) of resident records
        self.free_lists: dict = {}
        self.quarantine: list[int] = []
        self.qbytes = {sp: 0 for sp in SPACE_ORDER}
        self.next_id = 1                                 # campaign-scoped, not snapshotted
        self.dirty = {sp: set() for sp in SPACE_ORDER}
        self.sdirty = {sp: set() for sp in SPACE_ORDER}

    # address arithmetic -------------------------------------------------------
    def space_of(self, addr: int):
        for sp in SPACE_ORDER:
            if SPACE_BASE[sp] <= addr < SPACE_BASE[sp] + self.cfg.total(sp):
                return sp
        return None

    def _shade(self, sp, g0: int, n: int, code: int):
        if n <= 0:
            return
        self.shadow[sp][g0:g0 + n] = bytes([code]) * n
        self.sdirty[sp].update(range(g0 // CHUNK, (g0 + n - 1) // CHUNK + 1))

    def _poke(self, sp, off: int, data: bytes):
        if not data:
            return
        self.mem[sp][off:off + len(data)] = data
        self.dirty[sp].update(range(off // CHUNK, (off + len(data) - 1) // CHUNK + 1))

    def _paint(self, r: Rec, payload_code):
        g = self.cfg.granule
        b = SPACE_BASE[r.space]
        s0, p0 = (r.slot_start - b) // g, (r.base - b) // g
        p1, s1 = (_up(r.base + r.size, g) - b) // g, (r.slot_end - b) // g
        self._shade(r.space, s0, p0 - s0, SH_RZ)
        if payload_code is None:
            self._shade(r.space, p0, r.size // g, SH_OK)
            if r.size % g:
                self._shade(r.space, p0 + r.size // g, 1, r.size % g)
        else:
            self._shade(r.space, p0, p1 - p0, payload_code)
        self._shade(r.space, p1, s1 - p1, SH_RZ)

    # allocation ---------------------------------------------------------------
    def alloc(self, sp, size: int, label: str = "", scope: int = 0):
        c = self.cfg
        slot = c.redzone + _up(size, c.granule) + c.redzone
        key = (sp, scope, slot)
        bucket = self.free_lists.get(key)
        if bucket:
            off = bucket.pop(0)
            if not bucket:
                del self.free_lists[key]
        else:
            cur = self.cursor[(sp, scope)]
            end = (scope + 1) * c.scope_size(sp)
            if cur + slot > end:
                raise OutOfSpaceError(f"{sp.value} scope {scope}: need {slot} bytes, {end - cur} remain")
            off = cur
            self.cursor[(sp, scope)] = cur + slot
        start = SPACE_BASE[sp] + off
        r = Rec(self.next_id, sp, scope, start + c.redzone, size, "LIVE", label, start, start + slot)
        self.next_id += 1
        self.records[r.alloc_id] = r
        insort(self.rows[sp], (r.base, r.alloc_id))
        self._paint(r, None)
        self._poke(sp, r.base - SPACE_BASE[sp], bytes(size))
        return r.base, r.alloc_id

    def free(self, addr: int) -> int:
        sp = self.space_of(addr)
        if sp is None:
            raise InvalidFreeError(addr, "address outside all spaces")
        rows = self.rows[sp]
        i = bisect_right(rows, (addr, 1 << 62)) - 1
        if i < 0 or rows[i][0] != addr:
            raise InvalidFreeError(addr, "not the base of any resident allocation")
        r = self.records[rows[i][1]]
        if r.state == "FREED":
            raise InvalidFreeError(addr, "allocation already freed")
        r.state = "FREED"
        self._paint(r, SH_FREED)
        self.quarantine.append(r.alloc_id)
        self.qbytes[sp] += r.slot_end - r.slot_start
        while self.qbytes[sp] > self.cfg.qcap(sp):
            self._evict(sp)
        return r.alloc_id

    def _evict(self, sp):
        for qi, rid in enumerate(self.quarantine):
            if self.records[rid].space == sp:
                del self.quarantine[qi]
                r = self.records[rid]
                break
        else:
            raise AssertionError("quarantine accounting out of sync")
        g, b = self.cfg.granule, SPACE_BASE[sp]
        self._shade(sp, (r.slot_start - b) // g, (r.slot_end - r.slot_start) // g, SH_UNALLOC)
        self.rows[sp].remove((r.base, r.alloc_id))
        slot = r.slot_end - r.slot_start
        insort(self.free_lists.setdefault((sp, r.scope, slot), []), r.slot_start - b)
        self.qbytes[sp] -= slot

    # lookup -------------------------------------------------------------------
    def resolve_payload(self, addr: int):
        sp = self.space_of(addr)
        if sp is None:
            return None
        rows = self.rows[sp]
        i = bisect_right(rows, (addr, 1 << 62)) - 1
        if i < 0:
            return None
        r = self.records[rows[i][1]]
        return r if r.base <= addr < r.base + r.size else None

    def resolve_slot(self, addr: int):
        sp = self.space_of(addr)
        if sp is None:
            return None
        rows = self.rows[sp]
        i = bisect_right(rows, (addr, 1 << 62)) - 1
        for j in (i, i + 1):
            if 0 <= j < len(rows):
                r = self.records[rows[j][1]]
                if r.slot_start <= addr < r.slot_end:
                    return r
        return None

    def read(self, addr: int, n: int) -> bytes:
        sp = self.space_of(addr)
        off = addr - SPACE_BASE[sp]
        return bytes(self.mem[sp][off:off + n])

    def write(self, addr: int, data: bytes):
        sp = self.space_of(addr)
        self._poke(sp, addr - SPACE_BASE[sp], data)

    # host copies ---------------------------------------------------------------
    def copy_in(self, addr: int, data: bytes):
        if not data:
            return None
        rep = check_host(self, addr, len(data), True)
        if rep is None:
            self.write(addr, data)
        return rep

    def copy_out(self, addr: int, n: int):
        if n == 0:
            return b"", None
        rep = check_host(self, addr, n, False)
        return (None, rep) if rep is not None else (self.read(addr, n), None)

    # snapshot / restore --------------------------------------------------------
    def snapshot(self):
        snap = {
            "mem": {sp: bytes(self.mem[sp]) for sp in SPACE_ORDER},
            "shadow": {sp: bytes(self.shadow[sp]) for sp in SPACE_ORDER},
            "meta": copy.deepcopy((self.records, self.rows, self.cursor, self.free_lists,
                                   self.quarantine, self.qbytes)),
        }
        for sp in SPACE_ORDER:
            self.dirty[sp].clear()
            self.sdirty[sp].clear()
        return snap

    def restore(self, snap):
        for sp in SPACE_ORDER:
            for tbl, src, dirty in ((self.mem[sp], snap["mem"][sp], self.dirty[sp]),
                                    (self.shadow[sp], snap["shadow"][sp], self.sdirty[sp])):
                for ci in dirty:
                    tbl[ci * CHUNK:(ci + 1) * CHUNK] = src[ci * CHUNK:(ci + 1) * CHUNK]
                dirty.clear()
        (self.records, self.rows, self.cursor, self.free_lists, self.quarantine,
         self.qbytes) = copy.deepcopy(snap["meta"])


# -- classifier -------------------------------------------------------------------


def _fields(r):
    if r is None:
        return dict(alloc_id=None, alloc_label="", alloc_base=0, alloc_size=0, alloc_state="")
    return dict(alloc_id=r.alloc_id, alloc_label=r.label, alloc_base=r.base, alloc_size=r.size,
                alloc_state=r.state)


def scan_shadow(img: Image, addr: int, width: int):
    g = img.cfg.granule
    sp = img.space_of(addr)
    if sp is None:
        return ("wild", addr, SH_UNALLOC)
    sb = SPACE_BASE[sp]
    sh = img.shadow[sp]
    end = addr + width
    gi = (addr - sb) // g
    while sb + gi * g < end:
        if gi >= len(sh):
            return ("wild", sb + gi * g, SH_UNALLOC)
        code = sh[gi]
        if code != SH_OK:
            ga = sb + gi * g
            if code == SH_RZ:
                return ("spatial", ga, code)
            if code == SH_FREED:
                return ("freed", ga, code)
            if code == SH_UNALLOC:
                return ("wild", ga, code)
            lo = max(addr - sb, gi * g) - gi * g
            hi = min(end - sb, gi * g + g) - gi * g
            if lo >= code or hi > code:
                return ("spatial", ga, code)
        gi += 1
    return None


def check_access(img: Image, addr, width, space, prov, *, kernel, iid, ctaid=-1, tid=-1,
                 is_store=False, iteration=-1):
    def rep(cls, mech, shadow, rec):
        return BugReport(cls, kernel, iid, ctaid, tid, addr, width, is_store, space, mech, shadow,
                         prov, iteration=iteration, **_fields(rec))

    r = img.resolve_payload(addr)
    if r is not None and r.space != space:
        return rep(BugClass.SPACE_MISMATCH, "registry", None, r)
    if r is not None and r.state == "FREED":
        return rep(BugClass.TEMPORAL_UAF, "shadow", SH_FREED, r)
    v = scan_shadow(img, addr, width)
    if v is not None and v[0] == "spatial":
        return rep(BugClass.SPATIAL_OOB, "shadow", v[2], r if r is not None else img.resolve_slot(v[1]))
    if v is not None and v[0] == "freed":
        return rep(BugClass.TEMPORAL_UAF, "shadow", v[2], img.resolve_slot(v[1]))
    if prov is not None:
        t = img.records.get(prov)
        if t is not None and not (t.base <= addr and addr + width <= t.base + t.size):
            return rep(BugClass.PROVENANCE_ESCAPE, "provenance", v[2] if v else None, t)
    if v is not None:
        return rep(BugClass.WILD_ACCESS, "shadow", v[2], None)
    return None


def check_host(img: Image, addr, width, is_store, iteration=-1):
    return check_access(img, addr, width, img.space_of(addr) or MemSpace.GLOBAL, None,
                        kernel=HOST, iid=-1, is_store=is_store, iteration=iteration)


def invalid_free_report(img: Image, addr: int, iteration=-1):
    r = img.resolve_payload(addr) or img.resolve_slot(addr)
    return BugReport(BugClass.INVALID_FREE, HOST, -1, -1, -1, addr, 0, False, img.space_of(addr),
                     "registry", None, None, iteration=iteration, **_fields(r))
