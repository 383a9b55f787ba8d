"""Sanitizer report records and the deduplicated findings log (host types).

Classification itself runs on the GPU (``csrc/execute.cu``: ``check_access``);
the device emits a fixed-size verdict record per input which the host turns
into these objects only for inputs that open a new dedupe key.  Field meaning,
dedupe-key hashing and the text line follow the reference
``simt_forge/sanitizer.py:44-92`` (BugClass, BugReport) and ``:208-253``
(FindingsLog), so ``findings.txt`` renders byte-identically.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from enum import Enum

from .sir import MemSpace

HOST = "<host>"


class BugClass(Enum):
    SPATIAL_OOB = "SPATIAL_OOB"
    TEMPORAL_UAF = "TEMPORAL_UAF"
    SPACE_MISMATCH = "SPACE_MISMATCH"
    PROVENANCE_ESCAPE = "PROVENANCE_ESCAPE"
    WILD_ACCESS = "WILD_ACCESS"
    INVALID_FREE = "INVALID_FREE"


# device class codes (csrc/sfg_types.h SFG_CLASS_*) in this order
CLASS_BY_CODE = (BugClass.SPATIAL_OOB, BugClass.TEMPORAL_UAF, BugClass.SPACE_MISMATCH,
                 BugClass.PROVENANCE_ESCAPE, BugClass.WILD_ACCESS, BugClass.INVALID_FREE)
MECHANISMS = ("shadow", "registry", "provenance")


def dedupe_key_for(bug_class: BugClass, kernel: str, iid: int, site: str) -> str:
    return hashlib.sha256(f"{bug_class.value}|{kernel}|{iid}|{site}".encode()).hexdigest()[:16]


@dataclass
class BugReport:
    bug_class: BugClass
    kernel: str
    iid: int
    ctaid: int
    tid: int
    address: int
    width: int
    is_store: bool
    declared_space: MemSpace | None
    mechanism: str
    shadow_code: int | None
    provenance: int | None
    alloc_id: int | None
    alloc_label: str
    alloc_base: int
    alloc_size: int
    alloc_state: str
    iteration: int = -1
    dedupe_key: str = field(default="", compare=False)

    def __post_init__(self):
        if not self.dedupe_key:
            site = self.alloc_label if self.alloc_id is not None else "unmapped"
            self.dedupe_key = dedupe_key_for(self.bug_class, self.kernel, self.iid, site)

    def to_line(self) -> str:
        sp = self.declared_space.value if self.declared_space else "-"
        shadow = "-" if self.shadow_code is None else f"0x{self.shadow_code:02x}"
        return (f"finding class={self.bug_class.value} dedupe={self.dedupe_key} "
                f"kernel={self.kernel} iid={self.iid} ctaid={self.ctaid} tid={self.tid} "
                f"addr=0x{self.address:x} width={self.width} store={int(self.is_store)} "
                f"space={sp} mech={self.mechanism} shadow={shadow} "
                f"prov={'-' if self.provenance is None else self.provenance} "
                f"alloc={'-' if self.alloc_id is None else self.alloc_id} "
                f"label={self.alloc_label or '-'} base=0x{self.alloc_base:x} "
                f"size={self.alloc_size} state={self.alloc_state or '-'} "
                f"iteration={self.iteration}")


class FindingsLog:
    """Deduplicated findings in first-sighting order with per-key hit counts."""

    def __init__(self):
        self._order: list[str] = []
        self._first: dict[str, BugReport] = {}
        self._counts: dict[str, int] = {}

    def add(self, report: BugReport) -> bool:
        return self.add_many(report, 1)

    def add_many(self, report: BugReport, hits: int) -> bool:
        """Record ``hits`` sightings whose first one is ``report`` (batched
        absorption of one round).  True when the key is new."""
        key = report.dedupe_key
        if key in self._first:
            self._counts[key] += hits
            return False
        self._order.append(key)
        self._first[key] = report
        self._counts[key] = hits
        return True

    def bump(self, key: str, hits: int) -> None:
        self._counts[key] += hits

    def __contains__(self, key: str) -> bool:
        return key in self._first

    def __len__(self) -> int:
        return len(self._order)

    @property
    def total(self) -> int:
        return sum(self._counts.values())

    def reports(self) -> list[BugReport]:
        return [self._first[k] for k in self._order]

    def count(self, key: str) -> int:
        return self._counts.get(key, 0)

    def classes(self) -> set:
        return {r.bug_class for r in self._first.values()}

    def first_of_class(self, bug_class: BugClass) -> BugReport | None:
        for k in self._order:
            if self._first[k].bug_class == bug_class:
                return self._first[k]
        return None

    def render_text(self) -> str:
        rows = [f"unique={len(self._order)} total={self.total}"]
        rows += [self._first[k].to_line() + f" hits={self._counts[k]}" for k in self._order]
        return "\n".join(rows) + "\n"
