"""Harness manifests (.man): argspecs + INIT/COMPUTE/TERM host-op scripts.

Host-side, once per campaign.  Grammar, normalisation, digest and the static
semantic checks follow the reference ``simt_forge/campaign.py:83-389``
(HostOp, HarnessManifest, _parse_argspec, _parse_host_op, load_harness,
_validate_semantics) so that manifest digests and validation errors match.
The COMPUTE script is lowered to a device host-op table by :mod:`lowering`
and interpreted per fuzz input inside the execute kernel.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from pathlib import Path

from .sir import MemSpace, Program, ScalarType, parse_program, print_program, validate
from .testcase import ArgSpec, TestCase, seed_testcase

INIT = "init"
COMPUTE = "compute"
TERM = "term"


class ManifestError(Exception):
    pass


class ManifestSyntaxError(ManifestError):
    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


class UnknownKernelRefError(ManifestError):
    pass


class DanglingFreeError(ManifestError):
    pass


class ArgArityError(ManifestError):
    pass


@dataclass
class HostOp:
    kind: str
    line: int
    name: str = ""
    space: MemSpace | None = None
    size: int = 0
    source: tuple = ("", "")
    arg_ref: int = -1
    kernel: str = ""
    grid: int = 0
    block: int = 0
    bindings: tuple = ()


@dataclass
class HarnessManifest:
    path: Path
    program_path: Path
    program_text: str
    program: Program
    argspecs: list
    phases: dict
    normalized: str
    digest: str

    @property
    def program_digest(self) -> str:
        return self.program.digest

    def seed(self, rng_seed: int = 0) -> TestCase:
        return seed_testcase(self.argspecs, rng_seed)

    def portable_text(self, program_rel: str) -> str:
        lines = self.normalized.splitlines()
        lines[0] = f"program {program_rel}"
        return "\n".join(lines) + "\n"


_I32_LO = str(-(1 << 31))
_I32_HI = str((1 << 31) - 1)


def _argspec(toks: list, ln: int) -> ArgSpec:
    if len(toks) < 2:
        raise ManifestSyntaxError(ln, "argspec needs a name and a type")
    name, ty, rest = toks[0], toks[1], toks[2:]
    space = elem = None
    if ty == "ptr":
        if len(rest) < 2:
            raise ManifestSyntaxError(ln, "ptr argspec needs a space and element type")
        try:
            space = MemSpace(rest[0])
        except ValueError:
            raise ManifestSyntaxError(ln, f"unknown space {rest[0]!r}") from None
        elem = rest[1]
        if elem not in ("i32", "f32"):
            raise ManifestSyntaxError(ln, f"unknown element type {elem!r}")
        rest = rest[2:]
    kv, flags = {}, set()
    for t in rest:
        if "=" in t:
            k, _, v = t.partition("=")
            kv[k] = v
        else:
            flags.add(t)
    fixed = "fixed" in flags
    try:
        if ty == "i32":
            return ArgSpec(name, ScalarType.I32, seed_int=int(kv.get("seed", "0"), 0),
                           lo=int(kv.get("lo", _I32_LO), 0), hi=int(kv.get("hi", _I32_HI), 0),
                           fixed=fixed)
        if ty == "f32":
            return ArgSpec(name, ScalarType.F32, seed_float=float(kv.get("seed", "0")),
                           flo=float(kv.get("flo", "-1000")), fhi=float(kv.get("fhi", "1000")),
                           fixed=fixed)
        if ty == "ptr":
            count = int(kv["count"], 0)
            extents = tuple(int(t) for t in kv["extents"].split("x")) if "extents" in kv else (count,)
            seed = kv.get("seed", "zeros")
            fill, hexs, sf, si = "zeros", "", 0.0, 0
            if seed in ("zeros", "seq"):
                fill = seed
            elif seed.startswith("const:"):
                fill = "const"
                if elem == "f32":
                    sf = float(seed[6:])
                else:
                    si = int(seed[6:], 0)
            elif seed.startswith("hex:"):
                fill, hexs = "hex", seed[4:]
            else:
                raise ManifestSyntaxError(ln, f"unknown array seed {seed!r}")
            n = 1
            for e in extents:
                n *= e
            if n != count:
                raise ManifestSyntaxError(ln, "extents do not multiply to count")
            return ArgSpec(name, ScalarType.PTR, elem=elem, count=count, extents=extents,
                           space=space, seed_fill=fill, seed_hex=hexs, seed_float=sf, seed_int=si,
                           flo=float(kv.get("flo", "-1000")), fhi=float(kv.get("fhi", "1000")),
                           lo=int(kv.get("lo", _I32_LO), 0), hi=int(kv.get("hi", _I32_HI), 0),
                           fixed=fixed)
    except (KeyError, ValueError) as exc:
        raise ManifestSyntaxError(ln, f"bad argspec: {exc}") from None
    raise ManifestSyntaxError(ln, f"unknown argspec type {ty!r}")


def _binding(tok: str, ln: int) -> tuple:
    form, _, rest = tok.partition(":")
    if form == "arg":
        return ("arg", int(rest))
    if form == "buf":
        return ("buf", rest)
    if form == "lit":
        ty, _, lit = rest.partition(":")
        if ty == "i32":
            return ("lit_i32", int(lit, 0))
        if ty == "f32":
            return ("lit_f32", float(lit))
    raise ManifestSyntaxError(ln, f"bad launch binding {tok!r}")


def _host_op(line: str, ln: int) -> HostOp:
    t = line.split()
    kind = t[0]
    if kind == "alloc":
        if len(t) != 4:
            raise ManifestSyntaxError(ln, "alloc <name> <space> <bytes>")
        try:
            sp = MemSpace(t[2])
        except ValueError:
            raise ManifestSyntaxError(ln, f"unknown space {t[2]!r}") from None
        return HostOp("alloc", ln, name=t[1], space=sp, size=int(t[3], 0))
    if kind == "copy_in":
        if len(t) != 3:
            raise ManifestSyntaxError(ln, "copy_in <name> <source>")
        form, _, payload = t[2].partition(":")
        if form not in ("zeros", "seq32", "hex", "arg"):
            raise ManifestSyntaxError(ln, f"unknown copy_in source {t[2]!r}")
        return HostOp("copy_in", ln, name=t[1], source=(form, payload))
    if kind == "copy_out":
        if len(t) == 2 and t[1].startswith("arg:"):
            return HostOp("copy_out", ln, arg_ref=int(t[1][4:]))
        if len(t) == 3:
            return HostOp("copy_out", ln, name=t[1], size=int(t[2], 0))
        raise ManifestSyntaxError(ln, "copy_out arg:<k> | copy_out <name> <len>")
    if kind == "free":
        if len(t) != 2:
            raise ManifestSyntaxError(ln, "free <name>")
        return HostOp("free", ln, name=t[1])
    if kind == "launch":
        if len(t) < 2:
            raise ManifestSyntaxError(ln, "launch <kernel> grid=<n> block=<n> args=...")
        kv = dict(x.partition("=")[::2] for x in t[2:])
        try:
            b = tuple(_binding(x, ln) for x in kv["args"].split(",")) if kv.get("args") else ()
            return HostOp("launch", ln, kernel=t[1], grid=int(kv["grid"]), block=int(kv["block"]),
                          bindings=b)
        except (KeyError, ValueError) as exc:
            raise ManifestSyntaxError(ln, f"bad launch: {exc}") from None
    if kind == "sync":
        return HostOp("sync", ln)
    raise ManifestSyntaxError(ln, f"unknown host op {kind!r}")


def harness_from_text(text: str, program_text: str, path: Path | str = "harness.man",
                      program_path: Path | str | None = None) -> HarnessManifest:
    """Parse manifest text whose ``program`` line is resolved by the caller."""
    phases = {INIT: [], COMPUTE: [], TERM: []}
    specs: list = []
    section = None
    norm: list = []
    saw_program = False
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.endswith(":") and line[:-1] in phases:
            norm.append(line)
            section = line[:-1]
            continue
        t = line.split()
        if t[0] == "program":
            if len(t) != 2:
                raise ManifestSyntaxError(ln, "program <path>")
            saw_program = True
            continue
        norm.append(line)
        if t[0] == "argspec":
            if section is not None:
                raise ManifestSyntaxError(ln, "argspec must appear before phases")
            specs.append(_argspec(t[1:], ln))
            continue
        if section is None:
            raise ManifestSyntaxError(ln, f"{t[0]!r} outside any phase section")
        phases[section].append(_host_op(line, ln))
    if not saw_program:
        raise ManifestSyntaxError(0, "manifest names no program")
    program = parse_program(program_text)
    diags = validate(program)
    if diags:
        raise ManifestError(f"program has {len(diags)} diagnostics; first: {diags[0]}")
    if len({s.name for s in specs}) != len(specs):
        raise ManifestSyntaxError(0, "duplicate argspec names")
    _check(program, specs, phases)
    normalized = "\n".join([f"program sha256:{program.digest}"] + norm) + "\n"
    digest = hashlib.sha256(normalized.encode()).hexdigest()[:16]
    return HarnessManifest(Path(path), Path(program_path or "program.sir"), print_program(program),
                           program, specs, phases, normalized, digest)


def load_harness(path) -> HarnessManifest:
    path = Path(path)
    try:
        raw = path.read_text()
    except OSError as exc:
        raise ManifestError(f"cannot read manifest: {exc}") from exc
    rel = None
    for ln, rawline in enumerate(raw.splitlines(), start=1):
        t = rawline.split("#", 1)[0].split()
        if t and t[0] == "program" and len(t) == 2:
            rel = t[1]
    if rel is None:
        return harness_from_text(raw, "", path)  # raises the "names no program" error
    ppath = (path.parent / rel).resolve()
    try:
        src = ppath.read_text()
    except OSError as exc:
        raise ManifestError(f"cannot read program: {exc}") from exc
    return harness_from_text(raw, src, path, ppath)


def _check(program: Program, specs: list, phases: dict) -> None:
    arity = len(specs)
    used: set = set()

    def arg_ok(k: int, op: HostOp) -> None:
        if not 0 <= k < arity:
            raise ArgArityError(f"line {op.line}: arg:{k} outside argspec arity {arity}")
        used.add(k)

    init_bufs = {op.name for op in phases[INIT] if op.kind == "alloc"}
    known = {INIT: set(init_bufs)}
    known[COMPUTE] = init_bufs | {op.name for op in phases[COMPUTE] if op.kind == "alloc"}
    known[TERM] = set(known[COMPUTE])
    for phase, ops in phases.items():
        for op in ops:
            if op.kind in ("copy_in", "copy_out", "free") and op.name and op.name not in known[phase]:
                if op.kind == "free":
                    raise DanglingFreeError(f"line {op.line}: free of never-allocated {op.name!r}")
                raise ManifestSyntaxError(op.line, f"unknown buffer {op.name!r}")
            if op.kind == "copy_in" and op.source[0] == "arg":
                arg_ok(int(op.source[1]), op)
            if op.kind == "copy_out" and op.arg_ref >= 0:
                arg_ok(op.arg_ref, op)
            if op.kind != "launch":
                continue
            k = program.kernels.get(op.kernel)
            if k is None:
                raise UnknownKernelRefError(f"line {op.line}: kernel {op.kernel!r} not in program")
            if len(op.bindings) != len(k.params):
                raise ArgArityError(f"line {op.line}: {op.kernel} takes {len(k.params)} "
                                    f"params, {len(op.bindings)} bindings given")
            if op.grid < 1 or op.block < 1:
                raise ManifestSyntaxError(op.line, "grid and block must be >= 1")
            for b, p in zip(op.bindings, k.params):
                if b[0] == "arg":
                    arg_ok(b[1], op)
                    if specs[b[1]].kind != p.type:
                        raise ArgArityError(f"line {op.line}: arg:{b[1]} is {specs[b[1]].kind.value}, "
                                            f"param {p.name!r} wants {p.type.value}")
                elif b[0] == "buf":
                    if p.type != ScalarType.PTR:
                        raise ArgArityError(f"line {op.line}: buf binding on non-pointer param {p.name!r}")
                    if b[1] not in known[phase]:
                        raise ManifestSyntaxError(op.line, f"unknown buffer {b[1]!r}")
                elif b[0] == "lit_i32" and p.type != ScalarType.I32:
                    raise ArgArityError(f"line {op.line}: i32 literal on {p.type.value} param")
                elif b[0] == "lit_f32" and p.type != ScalarType.F32:
                    raise ArgArityError(f"line {op.line}: f32 literal on {p.type.value} param")
    if not any(op.kind == "launch" for op in phases[COMPUTE]):
        raise ManifestSyntaxError(0, "compute phase has no launch")
    frees = {op.name for op in phases[TERM] if op.kind == "free"}
    if init_bufs - frees:
        raise ManifestSyntaxError(0, f"term does not free: {sorted(init_bufs - frees)}")
    if frees - init_bufs:
        raise DanglingFreeError(f"term frees non-init buffers: {sorted(frees - init_bufs)}")
    if set(range(arity)) - used:
        raise ArgArityError(f"argspecs never referenced: {sorted(set(range(arity)) - used)}")
