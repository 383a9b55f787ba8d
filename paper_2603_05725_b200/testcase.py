"""Typed test cases, argument specs and mutation-op records (host data model).

These are the reference's public data types (``simt_forge/mutation.py``) so
that callers of the reference fuzz loop can hand the same objects to this
framework.  Nothing here mutates anything: the type-aware mutator itself runs
on the GPU (``csrc/mutate.cu``); the host only

* builds seed values from argspecs (reference ``seed_value`` mutation.py:163-185),
* packs test cases into the device corpus layout (:mod:`lowering`), and
* rebuilds ``TestCase`` objects from device records for admitted / crashing
  inputs, including the content-addressed id (mutation.py:234-248, 560-587).
"""

from __future__ import annotations

import ctypes
import hashlib
import struct
from dataclasses import dataclass, field

from .sir import MemSpace, ScalarType

I32_MAX = (1 << 31) - 1
I32_MIN = -(1 << 31)
F32_MAX_BITS = 0x7F7FFFFF
F32_MIN_BITS = 0xFF7FFFFF

TYPE_AWARE_KINDS = frozenset({
    "int_boundary", "float_sign", "float_exponent", "float_mantissa",
    "float_arith", "array_extreme", "array_dim", "array_empty",
    "ptr_space", "ptr_offset",
})
GENERIC_KINDS = frozenset({"int_byte", "float_byte", "array_elem"})


class MutationError(Exception):
    pass


def f32_round(v: float) -> float:
    """Round a python float to binary32 (inf on overflow), x86 host semantics."""
    return ctypes.c_float(v).value


def f32_bits(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", f32_round(v)))[0]


def bits_f32(b: int) -> float:
    return struct.unpack("<f", struct.pack("<I", b & 0xFFFFFFFF))[0]


@dataclass(frozen=True)
class IntValue:
    value: int

    def __post_init__(self):
        object.__setattr__(self, "value", ((self.value + (1 << 31)) & 0xFFFFFFFF) - (1 << 31))


@dataclass(frozen=True)
class FloatValue:
    bits: int

    def __post_init__(self):
        object.__setattr__(self, "bits", self.bits & 0xFFFFFFFF)

    @classmethod
    def from_float(cls, v: float) -> "FloatValue":
        return cls(f32_bits(v))

    @property
    def value(self) -> float:
        return bits_f32(self.bits)


@dataclass(frozen=True)
class ArrayValue:
    data: bytes
    elem: str
    extents: tuple
    space: MemSpace
    base_offset: int = 0
    size_override: int | None = None

    @property
    def count(self) -> int:
        n = 1
        for e in self.extents:
            n *= e
        return n


TypedValue = IntValue | FloatValue | ArrayValue


@dataclass(frozen=True)
class ArgSpec:
    name: str
    kind: ScalarType
    elem: str = "f32"
    count: int = 0
    extents: tuple = ()
    space: MemSpace = MemSpace.GLOBAL
    seed_int: int = 0
    seed_float: float = 0.0
    seed_fill: str = "zeros"
    seed_hex: str = ""
    lo: int = I32_MIN
    hi: int = I32_MAX
    flo: float = -1000.0
    fhi: float = 1000.0
    fixed: bool = False

    def canonical(self) -> str:
        if self.kind == ScalarType.I32:
            return f"{self.name} i32 seed={self.seed_int} lo={self.lo} hi={self.hi} fixed={int(self.fixed)}"
        if self.kind == ScalarType.F32:
            return (f"{self.name} f32 seed={self.seed_float!r} flo={self.flo!r} "
                    f"fhi={self.fhi!r} fixed={int(self.fixed)}")
        ext = "x".join(map(str, self.extents))
        return (f"{self.name} ptr {self.space.value} {self.elem} count={self.count} "
                f"extents={ext} fill={self.seed_fill} hex={self.seed_hex} "
                f"flo={self.flo!r} fhi={self.fhi!r} fixed={int(self.fixed)}")


def argspec_digest(specs) -> str:
    return hashlib.sha256("\n".join(s.canonical() for s in specs).encode()).hexdigest()[:16]


def seed_value(spec: ArgSpec) -> TypedValue:
    if spec.kind == ScalarType.I32:
        return IntValue(spec.seed_int)
    if spec.kind == ScalarType.F32:
        return FloatValue.from_float(spec.seed_float)
    n = spec.count
    if spec.seed_fill == "hex":
        data = bytes.fromhex(spec.seed_hex)
        if len(data) != 4 * n:
            raise MutationError(f"{spec.name}: hex seed length does not match count")
    elif spec.seed_fill == "seq":
        if spec.elem == "f32":
            data = b"".join(struct.pack("<I", f32_bits(float(i))) for i in range(n))
        else:
            data = b"".join(struct.pack("<i", i) for i in range(n))
    elif spec.seed_fill == "const":
        word = (struct.pack("<I", f32_bits(spec.seed_float)) if spec.elem == "f32"
                else struct.pack("<i", spec.seed_int))
        data = word * n
    else:
        data = bytes(4 * n)
    return ArrayValue(data, spec.elem, spec.extents or (n,), spec.space)


@dataclass(frozen=True)
class MutationOp:
    kind: str
    arg: int
    params: tuple = ()

    def param(self, key: str, default: str | None = None) -> str:
        for k, v in self.params:
            if k == key:
                return v
        if default is None:
            raise MutationError(f"{self.kind}: missing param {key!r}")
        return default

    def encode(self) -> str:
        return " ".join([f"mut {self.kind} arg={self.arg}"] + [f"{k}={v}" for k, v in self.params])

    @classmethod
    def make(cls, kind: str, arg: int, **params) -> "MutationOp":
        return cls(kind, arg, tuple(sorted((k, str(v)) for k, v in params.items())))

    @classmethod
    def decode(cls, line: str) -> "MutationOp":
        toks = line.split()
        if len(toks) < 3 or toks[0] != "mut":
            raise MutationError(f"bad mutation line: {line!r}")
        if toks[1] not in TYPE_AWARE_KINDS and toks[1] not in GENERIC_KINDS:
            raise MutationError(f"unknown mutation kind {toks[1]!r}")
        kv = dict(t.partition("=")[::2] for t in toks[2:])
        arg = int(kv.pop("arg"))
        return cls(toks[1], arg, tuple(sorted(kv.items())))

    @property
    def type_aware(self) -> bool:
        return self.kind in TYPE_AWARE_KINDS


@dataclass(frozen=True)
class TestCase:
    __test__ = False  # not a pytest class
    args: tuple
    rng_seed: int
    parent_id: str | None = None
    trace: tuple = ()
    _id: str = field(default="", compare=False)

    @property
    def id(self) -> str:
        if not self._id:
            body = serialize_testcase(self, with_id=False)
            object.__setattr__(self, "_id", hashlib.sha256(body.encode()).hexdigest()[:40])
        return self._id


def seed_testcase(specs, rng_seed: int = 0) -> TestCase:
    return TestCase(tuple(seed_value(s) for s in specs), rng_seed)


def _arg_line(i: int, v) -> str:
    if isinstance(v, IntValue):
        return f"arg{i} i32 value={v.value}"
    if isinstance(v, FloatValue):
        return f"arg{i} f32 bits=0x{v.bits:08x}"
    ov = "-" if v.size_override is None else str(v.size_override)
    return (f"arg{i} array elem={v.elem} space={v.space.value} extents={'x'.join(map(str, v.extents))} "
            f"offset={v.base_offset} override={ov} data={v.data.hex() or '-'}")


def serialize_testcase(tc: TestCase, specs=None, with_id: bool = True, extra=None) -> str:
    out = ["simt-forge-testcase v1"]
    if with_id:
        out.append(f"id={tc.id}")
    if specs is not None:
        out.append(f"argspec={argspec_digest(specs)}")
    out.append(f"rng_seed={tc.rng_seed}")
    out.append(f"parent={tc.parent_id or '-'}")
    out.extend(op.encode() for op in tc.trace)
    out.extend(_arg_line(i, v) for i, v in enumerate(tc.args))
    out.extend(extra or ())
    out.append("end")
    return "\n".join(out) + "\n"


def parse_testcase(text: str, specs=None):
    lines = [l for l in text.splitlines() if l.strip()]
    if not lines or lines[0] != "simt-forge-testcase v1":
        raise MutationError("not a testcase record")
    meta, trace, args, extra = {}, [], {}, {}
    for line in lines[1:]:
        if line == "end":
            break
        if line.startswith("mut "):
            trace.append(MutationOp.decode(line))
            continue
        head, _, rest = line.partition(" ")
        if head.startswith("arg") and head[3:].isdigit():
            kind, _, kvtext = rest.partition(" ")
            kv = dict(t.split("=", 1) for t in kvtext.split())
            if kind == "i32":
                args[int(head[3:])] = IntValue(int(kv["value"]))
            elif kind == "f32":
                args[int(head[3:])] = FloatValue(int(kv["bits"], 0))
            else:
                ext = tuple(int(t) for t in kv["extents"].split("x")) if kv["extents"] else (0,)
                args[int(head[3:])] = ArrayValue(
                    b"" if kv["data"] == "-" else bytes.fromhex(kv["data"]), kv["elem"], ext,
                    MemSpace(kv["space"]), int(kv["offset"]),
                    None if kv["override"] == "-" else int(kv["override"]))
            continue
        key, _, value = line.partition("=")
        if key in ("id", "argspec", "rng_seed", "parent"):
            meta[key] = value
        else:
            extra[line.split()[0]] = line
    if specs is not None and "argspec" in meta and meta["argspec"] != argspec_digest(specs):
        raise MutationError("testcase argspec digest does not match the harness")
    if sorted(args) != list(range(len(args))):
        raise MutationError("argument indices are not dense")
    parent = meta.get("parent", "-")
    tc = TestCase(tuple(args[i] for i in sorted(args)), int(meta.get("rng_seed", "0")),
                  None if parent == "-" else parent, tuple(trace))
    if "id" in meta and meta["id"] != tc.id:
        raise MutationError("testcase id does not match its content")
    return tc, extra


# ---- seed corpora ------------------------------------------------------------------------


class Stream:
    """Keyed random stream with the reference's semantics (rng.py:20-117: numpy's
    ``Generator`` over ``Philox`` keyed ``(seed, stream_id)``).  Host-side only
    (seed corpora); the device restates the same generator in csrc/philox.cuh."""

    def __init__(self, seed: int, stream_id: int = 0):
        import numpy as np
        self._gen = np.random.Generator(np.random.Philox(
            key=np.array([seed & 0xFFFFFFFFFFFFFFFF, stream_id & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)))

    def integers(self, lo: int, hi: int) -> int:
        return int(self._gen.integers(lo, hi))

    def random(self) -> float:
        return float(self._gen.random())

    def u64(self) -> int:
        import numpy as np
        return int(self._gen.integers(0, 1 << 64, dtype=np.uint64))


def sample_valid_testcase(specs, rng: Stream) -> TestCase:
    """Uniform draw from every argument's declared valid domain, draw for draw
    as the reference (mutation.py:533-554); used to build large seed corpora
    (BASELINE.json configs[3])."""
    import struct
    args = []
    for spec in specs:
        if spec.kind == ScalarType.I32:
            args.append(IntValue(rng.integers(spec.lo, spec.hi + 1)))
        elif spec.kind == ScalarType.F32:
            args.append(FloatValue.from_float(spec.flo + rng.random() * (spec.fhi - spec.flo)))
        else:
            if spec.elem == "f32":
                span = spec.fhi - spec.flo
                data = b"".join(struct.pack("<I", f32_bits(spec.flo + rng.random() * span))
                                for _ in range(spec.count))
            else:
                data = b"".join(struct.pack("<i", rng.integers(spec.lo, spec.hi + 1)) for _ in range(spec.count))
            args.append(ArrayValue(data, spec.elem, spec.extents or (spec.count,), spec.space))
    return TestCase(tuple(args), rng.u64())
