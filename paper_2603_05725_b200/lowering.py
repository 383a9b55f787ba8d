"""Lowering: harness manifest -> packed device tables, and record codecs.

Host-side, once per campaign (the analogue of the paper's instrument-at-load
step).  Produces the byte images of the structs in ``csrc/sfg_types.h``:

* ``sfg_ins``      one pre-decoded instruction; immediates prepared exactly as
                   the reference consumes them (``executor.py:257-362``:
                   i32 wrap, ``f32(float(imm))``, cvt of immediates folded)
* ``sfg_hostop`` / ``sfg_binding``  the COMPUTE host-op script (campaign.py:483-561)
* ``sfg_rec`` + baseline blob        post-INIT allocation state and payloads
                                     (built by :mod:`baseline`)
* ``sfg_prog``     scalar header passed by value to every kernel

and the codecs between host objects (``TestCase``, ``MutationOp``,
``BugReport``) and device records (``sfg_val``, ``sfg_op``, ``sfg_verdict``).
"""

from __future__ import annotations

import math
import struct

import numpy as np

from .findings import CLASS_BY_CODE, HOST, MECHANISMS, BugReport
from .manifest import COMPUTE
from .sir import SPACE_INDEX, SPACE_ORDER, MemSpace, Opcode, ScalarType
from .testcase import (ArrayValue, FloatValue, IntValue, MutationOp, TestCase, f32_bits)

MAX_ARGS = 16
MAX_OPS = 3
MAX_KERNELS = 16
MAX_NAMED = 32
MAX_BASE_RECS = 32
MAX_FREE = 32
MAX_REGS = 64
MAX_EDGES = 1024
MAX_LANE_RECS = 40   # sfg_types.h SFG_MAX_LANE_RECS: baseline + one input's own allocation records
MAX_QUAR = 32        # exec_core.cuh kMaxQ / kMaxFree: one input's quarantine and free list
NO_OVERRIDE = -(1 << 63)

# ---- struct dtypes (mirror csrc/sfg_types.h; sizes checked against the .so) ----

INS = np.dtype([("op", "u1"), ("mode", "u1"), ("flags", "u1"), ("dst", "u1"), ("s1", "u1"), ("s2", "u1"),
                ("space", "u1"), ("width", "u1"), ("target", "<i4"), ("edge_ft", "<i2"), ("edge_tk", "<i2"),
                ("imm1", "<i8"), ("imm2", "<i8")], align=True)
KERNEL = np.dtype([("ins_base", "<i4"), ("n_ins", "<i4"), ("regs", "<i4"), ("n_params", "<i4"),
                   ("edge_base", "<i4"), ("n_edges", "<i4"), ("n_blocks", "<i4"), ("name_idx", "<i4"),
                   ("ptype", "u1", (16,))], align=True)
HOSTOP = np.dtype([("kind", "<i4"), ("buf", "<i4"), ("space", "<i4"), ("kernel", "<i4"), ("size", "<i8"),
                   ("src_form", "<i4"), ("src_arg", "<i4"), ("blob_off", "<i8"), ("arg_ref", "<i4"),
                   ("grid", "<i4"), ("block", "<i4"), ("bind_base", "<i4"), ("n_bind", "<i4"),
                   ("label", "<i4"), ("work_off", "<i4"), ("pad", "<i4")], align=True)
BINDING = np.dtype([("form", "<i4"), ("idx", "<i4"), ("lit", "<i8")], align=True)
REC = np.dtype([("base", "<i8"), ("size", "<i8"), ("slot_start", "<i8"), ("slot_end", "<i8"), ("phys", "<i8"),
                ("id", "<i4"), ("label", "<i2"), ("space", "u1"), ("state", "u1"), ("resident", "u1"),
                ("scope", "u1"), ("pad", "u1", (14,))], align=True)
FREE = np.dtype([("off", "<i8"), ("slot", "<i8"), ("space", "<i4"), ("scope", "<i4")], align=True)
NAMED = np.dtype([("addr", "<i8"), ("id", "<i4"), ("rec", "<i4")], align=True)
VAL = np.dtype([("kind", "u1"), ("elem", "u1"), ("space", "u1"), ("ndim", "u1"), ("bits", "<u4"),
                ("data_off", "<u8"), ("nbytes", "<u4"), ("count", "<u4"), ("base_offset", "<i8"),
                ("size_override", "<i8"), ("ext", "<u4", (4,)), ("pad", "<u8")], align=True)
OP = np.dtype([("kind", "u1"), ("arg", "u1"), ("sub", "u1"), ("byte", "u1"), ("inner", "u1"), ("isub", "u1"),
               ("ibyte", "u1"), ("pad", "u1"), ("mask", "<u4"), ("imask", "<u4"), ("index", "<u4"),
               ("pad2", "<u4"), ("delta", "<i8")], align=True)
CHILD = np.dtype([("rng_seed", "<u8"), ("it", "<i8"), ("parent", "<i4"), ("n_ops", "<i4"),
                  ("work_bytes", "<u8"), ("readout_bytes", "<u8"), ("pad", "<u8"), ("ops", OP, (MAX_OPS,))],
                 align=True)
ENTRY = np.dtype([("admitted_iteration", "<i8"), ("rng_seed", "<u8"), ("is_seed", "<i4"), ("parent", "<i4"),
                  ("it", "<i8")], align=True)
VERDICT = np.dtype([("status", "<i4"), ("bug_class", "<i4"), ("kernel", "<i4"), ("iid", "<i4"),
                    ("ctaid", "<i4"), ("tid", "<i4"), ("width", "<i4"), ("shadow", "<i4"),
                    ("addr_lo", "<i8"), ("addr_hi", "<i8"), ("is_store", "u1"), ("space", "u1"), ("mech", "u1"),
                    ("alloc_state", "u1"), ("prov", "<i4"), ("alloc", "<i4"), ("label", "<i4"),
                    ("alloc_base", "<i8"), ("alloc_size", "<i8"), ("retired", "<u8"), ("launches", "<i4"),
                    ("allocs", "<i4"), ("entered", "<u4"), ("key", "<i4"), ("where", "<u8")], align=True)
PROG = np.dtype([
    ("space_size", "<i8", (3,)), ("scope_size", "<i8", (3,)), ("qcap", "<i8", (3,)),
    ("granule", "<i4"), ("redzone", "<i4"), ("cursor", "<i8", (3,)), ("qbytes", "<i8", (3,)),
    ("n_base_recs", "<i4"), ("n_free", "<i4"), ("n_quar", "<i4"), ("n_named", "<i4"),
    ("quar", "<i4", (MAX_BASE_RECS,)), ("named", NAMED, (MAX_NAMED,)), ("freel", FREE, (MAX_FREE,)),
    ("n_args", "<i4"), ("n_mutable", "<i4"), ("n_int_args", "<i4"), ("n_kernels", "<i4"),
    ("arg_kind", "u1", (MAX_ARGS,)), ("arg_elem", "u1", (MAX_ARGS,)), ("arg_fixed", "u1", (MAX_ARGS,)),
    ("mutable_args", "i1", (MAX_ARGS,)), ("int_slot", "i1", (MAX_ARGS,)),
    ("n_hostops", "<i4"), ("n_edges", "<i4"), ("n_labels", "<i4"), ("n_keys", "<i4"),
    ("label_arg_base", "<i4"), ("total_ins", "<i4"), ("named_work_bytes", "<i4"), ("ov_cap", "<i4"),
    ("kernels", KERNEL, (MAX_KERNELS,)),
    ("max_ops", "<i4"), ("mut_granule", "<i4"), ("mut_redzone", "<i4"), ("window", "<i4"),
    ("recent_weight", "<f8"), ("master_seed", "<u8"), ("keybase", "<u8"), ("budget", "<u8"),
    ("diff_readback", "<i4"), ("stop_first", "<i4"), ("stop_class", "<i4"), ("n_copyout_arg", "<i4"),
    ("readout_bytes_fixed", "<i8"), ("copyout_arg", "i1", (MAX_ARGS,)), ("fanout", "<i4"),
    ("copy_src_mask", "<u4"), ("term_phase", "<i4"), ("jit_off", "<i4")], align=True)

LAYOUTS = {"ins": INS, "kernel": KERNEL, "hostop": HOSTOP, "binding": BINDING, "rec": REC, "val": VAL,
           "op": OP, "child": CHILD, "entry": ENTRY, "verdict": VERDICT, "prog": PROG}

# enums (csrc/sfg_types.h)
CLS = {"r": 0, "f": 1, "a": 2, "p": 3}
CMP = {"eq": 0, "ne": 1, "lt": 2, "le": 3, "gt": 4, "ge": 5}
MK = {"b8": 0, "b16": 1, "b32": 2, "b64": 3, "f32": 4}
SREG = {"tid": 0, "ntid": 1, "ctaid": 2, "nctaid": 3}
F_S1_IMM, F_S2_IMM, F_PRED, F_PNEG, F_FLOAT, F_U64IMM = 0x01, 0x02, 0x04, 0x08, 0x10, 0x20
H_ALLOC, H_COPY_IN, H_COPY_OUT_NAMED, H_COPY_OUT_ARG, H_FREE, H_LAUNCH, H_SYNC = range(7)
SRC = {"zeros": 0, "seq32": 1, "hex": 2, "arg": 3}
B_ARG, B_BUF, B_LIT_I32, B_LIT_F32 = range(4)
V_I32, V_F32, V_ARR = range(3)
ST_OK, ST_FINDING, ST_BUDGET = 0, 1, 2
ST_OUT_OF_SPACE, ST_ZERO_ALLOC, ST_LANE_RECS, ST_OVERLAY, ST_COUNTER = 16, 17, 18, 19, 20
KEYBASE = 1 << 32

M_KINDS = ("int_boundary", "int_byte", "float_sign", "float_exponent", "float_mantissa", "float_byte",
           "float_arith", "array_extreme", "array_dim", "array_empty", "ptr_space", "ptr_offset", "array_elem")
M_INDEX = {k: i for i, k in enumerate(M_KINDS)}


from .baseline import LoweringError  # noqa: E402,F401  (the harness uses a construct this path does not lower)


OV_CHUNK = 256    # sfg_types.h SFG_OV_CHUNK
OV_CAP0 = 4       # initial overlay chunks per input of a harness that can write INIT buffers


def ov_bytes(cap: int) -> int:
    """Bytes of the copy-on-write overlay at the tail of a work region (sfg_ov_bytes)."""
    return 0 if cap <= 0 else ((cap * 8 + 15) & ~15) + cap * OV_CHUNK


def wrap_i32(v: int) -> int:
    return ((v + (1 << 31)) & 0xFFFFFFFF) - (1 << 31)


def cvt_f32_to_i32(v: float) -> int:   # executor.py:51-65
    if math.isnan(v):
        return 0
    if v >= 2147483647.0:
        return 2147483647
    if v <= -2147483648.0:
        return -2147483648
    f = math.floor(v)
    d = v - f
    if d > 0.5 or (d == 0.5 and f % 2):
        f += 1
    return int(f)


def _i64(v: int, what: str) -> int:
    if not -(1 << 63) <= v < (1 << 63):
        raise LoweringError(f"{what} immediate {v} does not fit in 64 bits")
    return v


# ---- instructions -------------------------------------------------------------------


def edge_table(program):
    """Dense global edge ids: kernels in program order, each kernel's sorted static edges."""
    ids, base = {}, 0
    per_kernel = {}
    for name, k in program.kernels.items():
        per_kernel[name] = base
        for j, e in enumerate(sorted(k.edges)):
            ids[(name, e)] = base + j
        base += len(k.edges)
    return ids, per_kernel, base


def lower_instructions(program):
    eids, ebase, n_edges = edge_table(program)
    if n_edges > MAX_EDGES:
        raise LoweringError(f"{n_edges} static edges exceed {MAX_EDGES}")
    rows = []
    kernels = []
    for kidx, (name, k) in enumerate(program.kernels.items()):
        if k.register_count > MAX_REGS:
            raise LoweringError(f"kernel {name}: regs={k.register_count} exceeds {MAX_REGS}")
        if len(k.params) > MAX_ARGS:
            raise LoweringError(f"kernel {name}: more than {MAX_ARGS} params")
        kernels.append(dict(ins_base=len(rows), n_ins=len(k.instructions), regs=k.register_count,
                            n_params=len(k.params), edge_base=ebase[name], n_edges=len(k.edges),
                            n_blocks=len(k.blocks), name_idx=kidx,
                            ptype=[{"i32": 0, "f32": 1, "ptr": 2}[p.type.value] for p in k.params]))
        ins = k.instructions
        for i in ins:
            rows.append(_lower_one(name, k, i, ins, eids))
    arr = np.zeros(len(rows), INS)
    for j, r in enumerate(rows):
        for key, v in r.items():
            arr[j][key] = v
    return arr, kernels, n_edges


def _lower_one(kname, k, i, ins, eids):
    r = dict(op=int(i.opcode), mode=0, flags=0, dst=0, s1=0, s2=0, space=0, width=0, target=0,
             edge_ft=-1, edge_tk=-1, imm1=0, imm2=0)
    op = i.opcode
    nxt = i.iid + 1
    if op not in (Opcode.BRA, Opcode.EXIT) and nxt < len(ins) and ins[nxt].block != i.block:
        r["edge_ft"] = eids[(kname, (i.block, ins[nxt].block))]

    def src(slot: int, operand, prep):
        if isinstance(operand, tuple):
            r["s1" if slot == 1 else "s2"] = operand[1]
        else:
            r["flags"] |= F_S1_IMM if slot == 1 else F_S2_IMM
            r["imm1" if slot == 1 else "imm2"] = prep(operand)

    def fimm(v):
        return f32_bits(float(v))

    if op == Opcode.MOV:
        c = i.dst[0]
        r["mode"], r["dst"] = CLS[c], i.dst[1]
        s = i.srcs[0]
        if c == "a" and not isinstance(s, tuple):
            v = int(s)
            if (1 << 63) <= v < (1 << 64):
                r["flags"] |= F_S1_IMM | F_U64IMM
                r["imm1"] = v - (1 << 64)
            else:
                r["flags"] |= F_S1_IMM
                r["imm1"] = _i64(v, "mov")
        else:
            src(1, s, (lambda v: wrap_i32(int(v))) if c == "r" else fimm)
    elif op in (Opcode.ADD, Opcode.SUB, Opcode.MUL):
        c = i.dst[0]
        r["mode"], r["dst"] = CLS[c], i.dst[1]
        if c == "a":
            r["s1"] = i.srcs[0][1]
            src(2, i.srcs[1], lambda v: _i64(int(v), "pointer add"))
        else:
            src(1, i.srcs[0], lambda v: wrap_i32(int(v)))
            src(2, i.srcs[1], lambda v: wrap_i32(int(v)))
    elif op in (Opcode.FADD, Opcode.FSUB, Opcode.FMUL):
        r["dst"] = i.dst[1]
        src(1, i.srcs[0], fimm)
        src(2, i.srcs[1], fimm)
    elif op == Opcode.SETP:
        r["mode"], r["dst"] = CMP[i.cmp], i.dst[1]
        is_f = any((isinstance(s, tuple) and s[0] == "f") or isinstance(s, float) for s in i.srcs)
        if is_f:
            r["flags"] |= F_FLOAT
            src(1, i.srcs[0], fimm)
            src(2, i.srcs[1], fimm)
        else:
            clamp = lambda v: max(-(1 << 63), min((1 << 63) - 1, int(v)))  # noqa: E731
            src(1, i.srcs[0], clamp)
            src(2, i.srcs[1], clamp)
    elif op == Opcode.BRA:
        r["target"] = i.target_iid
        if i.pred is not None:
            r["flags"] |= F_PRED | (F_PNEG if i.pred_negate else 0)
            r["s1"] = i.pred[1]
        r["edge_tk"] = eids[(kname, (i.block, ins[i.target_iid].block))]
        if nxt < len(ins):
            r["edge_ft"] = eids.get((kname, (i.block, ins[nxt].block)), -1)
    elif op in (Opcode.LD, Opcode.ST):
        base, off = i.addr
        r["space"], r["width"], r["mode"] = SPACE_INDEX[i.space], i.width, MK[i.mem_kind]
        r["s1"] = base[1]
        r["imm2"] = _i64(off, "address offset")
        if op == Opcode.LD:
            r["dst"] = i.dst[1]
        else:
            s = i.srcs[0]
            kind = i.mem_kind
            if isinstance(s, tuple):
                r["s2"] = s[1]
            else:
                r["flags"] |= F_S2_IMM
                if kind == "f32":
                    r["imm1"] = f32_bits(float(s))
                elif kind == "b32":
                    r["imm1"] = wrap_i32(int(s))
                elif kind == "b16":
                    r["imm1"] = int(s) & 0xFFFF
                elif kind == "b8":
                    r["imm1"] = int(s) & 0xFF
                else:
                    raise LoweringError("st.b64 needs a register source")
    elif op == Opcode.CVT:
        r["dst"] = i.dst[1]
        s = i.srcs[0]
        to_f = i.cvt[0] == ScalarType.F32
        r["mode"] = 0 if to_f else 1
        if isinstance(s, tuple):
            r["s1"] = s[1]
        else:
            r["flags"] |= F_S1_IMM
            r["imm1"] = f32_bits(float(int(s))) if to_f else cvt_f32_to_i32(float(s))
    elif op == Opcode.SREG:
        r["mode"], r["dst"] = SREG[i.sreg], i.dst[1]
    return r


# ---- host-op script -----------------------------------------------------------------


class Lowered:
    """Everything the device needs for one harness + campaign configuration."""

    def __init__(self, manifest, baseline, *, mem, mutation, master_seed, budget, window, recent_weight,
                 diff_readback=False, stop_first=False, stop_class=None, fanout=0, term_phase=False,
                 jit=True):
        self.manifest = manifest
        prog = manifest.program
        specs = manifest.argspecs
        if len(specs) > MAX_ARGS:
            raise LoweringError(f"more than {MAX_ARGS} argspecs")
        if len(prog.kernels) > MAX_KERNELS:
            raise LoweringError(f"more than {MAX_KERNELS} kernels")
        self.kernel_names = list(prog.kernels)
        self.ins, kernels, self.n_edges = lower_instructions(prog)
        self.edge_names = []
        for name, k in prog.kernels.items():
            self.edge_names += [(name, e) for e in sorted(k.edges)]
        # labels: named buffers (INIT + COMPUTE) then argK
        names = []
        for ph in ("init", "compute", "term"):
            for op in manifest.phases[ph]:
                if op.kind == "alloc" and op.name not in names:
                    names.append(op.name)
        if len(names) > MAX_NAMED:
            raise LoweringError("too many named buffers")
        self.buf_index = {n: j for j, n in enumerate(names)}
        self.labels = names + [f"arg{k}" for k in range(len(specs))]
        self.label_arg_base = len(names)
        total_ins = len(self.ins)
        self.total_ins = total_ins
        self.n_keys = 6 * (total_ins + 1) * (len(self.labels) + 1)
        self.baseline = baseline
        # COMPUTE script
        hops, binds = [], []
        const_blob = bytearray()
        named_work = 0
        self.copy_src_mask = 0      # array args that are COMPUTE copy_in sources
        copyout_args = []
        readout_fixed = 0
        for op in manifest.phases[COMPUTE]:
            h = dict(kind=0, buf=-1, space=0, kernel=-1, size=0, src_form=0, src_arg=-1, blob_off=0, arg_ref=-1,
                     grid=0, block=0, bind_base=0, n_bind=0, label=-1, work_off=0, pad=0)
            if op.kind == "alloc":
                h.update(kind=H_ALLOC, buf=self.buf_index[op.name], space=SPACE_INDEX[op.space], size=op.size,
                         label=self.buf_index[op.name], work_off=named_work)
                named_work += (max(op.size, 0) + 15) // 16 * 16
            elif op.kind == "copy_in":
                form, payload = op.source
                h.update(kind=H_COPY_IN, buf=self.buf_index[op.name], src_form=SRC[form])
                if form == "zeros":
                    h["size"] = int(payload, 0)
                elif form == "seq32":
                    h["size"] = 4 * int(payload, 0)
                elif form == "hex":
                    data = bytes.fromhex(payload)
                    h.update(size=len(data), blob_off=len(const_blob))
                    const_blob += data
                else:
                    k = int(payload)
                    # an array source copies the test case's own bytes (campaign.py:404-409,
                    # 497-513): the work region keeps a pristine copy of that argument
                    if specs[k].kind == ScalarType.PTR:
                        self.copy_src_mask |= 1 << k
                    h.update(src_arg=k, size=4)
            elif op.kind == "copy_out":
                if op.arg_ref >= 0:
                    h.update(kind=H_COPY_OUT_ARG, arg_ref=op.arg_ref)
                    if specs[op.arg_ref].kind == ScalarType.PTR:
                        copyout_args.append(op.arg_ref)
                else:
                    h.update(kind=H_COPY_OUT_NAMED, buf=self.buf_index[op.name], size=op.size)
                    readout_fixed += (max(op.size, 0) + 15) // 16 * 16
            elif op.kind == "free":
                h.update(kind=H_FREE, buf=self.buf_index[op.name])
            elif op.kind == "launch":
                h.update(kind=H_LAUNCH, kernel=self.kernel_names.index(op.kernel), grid=op.grid, block=op.block,
                         bind_base=len(binds), n_bind=len(op.bindings))
                for b in op.bindings:
                    if b[0] == "arg":
                        binds.append((B_ARG, b[1], 0))
                    elif b[0] == "buf":
                        binds.append((B_BUF, self.buf_index[b[1]], 0))
                    elif b[0] == "lit_i32":
                        binds.append((B_LIT_I32, 0, wrap_i32(int(b[1]))))
                    else:
                        binds.append((B_LIT_F32, 0, f32_bits(float(b[1]))))
            else:
                h.update(kind=H_SYNC)
            hops.append(h)
        self.hostops = np.zeros(max(len(hops), 1), HOSTOP)
        for j, h in enumerate(hops):
            for key, v in h.items():
                self.hostops[j][key] = v
        self.n_hostops = len(hops)
        self.binds = np.zeros(max(len(binds), 1), BINDING)
        for j, (f, ix, lit) in enumerate(binds):
            self.binds[j] = (f, ix, lit)
        self.const_blob = bytes(const_blob) or b"\0"
        # overlay needed when INIT buffers are reachable without a finding
        untagged = any(i.opcode == Opcode.MOV and i.dst[0] == "a" and not isinstance(i.srcs[0], tuple)
                       or (i.opcode == Opcode.LD and i.mem_kind == "b64")
                       for k in prog.kernels.values() for i in k.instructions)
        buf_bound = any(b[0] == "buf" for op in manifest.phases[COMPUTE] if op.kind == "launch" for b in op.bindings)
        init_copy = any(op.kind == "copy_in" and op.name not in
                        {o.name for o in manifest.phases[COMPUTE] if o.kind == "alloc"}
                        for op in manifest.phases[COMPUTE])
        self.overlay = bool(untagged or buf_bound or init_copy)
        # per-input table capacities, checked here at load time: an input allocates at
        # most one record per array argument (materialized once per phase,
        # campaign.py:440-450) and per COMPUTE alloc, and frees at most once per free op
        n_allocs = sum(1 for s in specs if s.kind == ScalarType.PTR) + \
            sum(1 for op in manifest.phases[COMPUTE] if op.kind == "alloc")
        n_frees = sum(1 for op in manifest.phases[COMPUTE] if op.kind == "free")
        if len(baseline.records) + n_allocs > MAX_LANE_RECS:
            raise LoweringError(f"INIT records + per-input allocations ({len(baseline.records)} + {n_allocs}) "
                                f"exceed the per-input table ({MAX_LANE_RECS})")
        if len(baseline.quarantine) + n_frees > MAX_QUAR or \
                len(baseline.free_entries) + len(baseline.quarantine) + n_frees > MAX_QUAR:
            raise LoweringError(f"quarantine / free list of an input can exceed {MAX_QUAR} entries")
        # header
        P = np.zeros(1, PROG)[0]
        for s, sp in enumerate(SPACE_ORDER):
            P["space_size"][s] = mem.scope_size(sp) * mem.scopes(sp)
            P["scope_size"][s] = mem.scope_size(sp)
            P["qcap"][s] = mem.qcap(sp)
            P["cursor"][s] = baseline.cursor[sp]
            P["qbytes"][s] = baseline.qbytes[sp]
        P["granule"], P["redzone"] = mem.granule, mem.redzone
        P["n_base_recs"] = len(baseline.records)
        P["n_free"] = len(baseline.free_entries)
        P["n_quar"] = len(baseline.quarantine)
        for j, ri in enumerate(baseline.quarantine):
            P["quar"][j] = ri
        for j, (off, slot, sp) in enumerate(baseline.free_entries):
            P["freel"][j] = (off, slot, SPACE_INDEX[sp], 0)
        P["n_named"] = len(names)
        for n, j in self.buf_index.items():
            if n in baseline.named:
                addr, aid, ri = baseline.named[n]
                P["named"][j] = (addr, aid, ri)
            else:
                P["named"][j] = (0, 0, -1)
        P["n_args"] = len(specs)
        mutable = [j for j, s in enumerate(specs) if not s.fixed]
        ints = [j for j, s in enumerate(specs) if s.kind == ScalarType.I32]
        P["n_mutable"], P["n_int_args"], P["n_kernels"] = len(mutable), len(ints), len(kernels)
        self.int_args = ints
        P["int_slot"][:] = -1
        for j, s in enumerate(specs):
            P["arg_kind"][j] = {ScalarType.I32: V_I32, ScalarType.F32: V_F32, ScalarType.PTR: V_ARR}[s.kind]
            P["arg_elem"][j] = 1 if s.elem == "f32" else 0
            P["arg_fixed"][j] = int(s.fixed)
        for j, a in enumerate(mutable):
            P["mutable_args"][j] = a
        for c, a in enumerate(ints):
            P["int_slot"][a] = c
        P["n_hostops"], P["n_edges"], P["n_labels"], P["n_keys"] = len(hops), self.n_edges, len(self.labels), self.n_keys
        P["label_arg_base"], P["total_ins"], P["named_work_bytes"] = self.label_arg_base, total_ins, named_work
        # copy-on-write overlay chunks per input (grown by the engine when a round
        # overflows it; the round is then re-run, so no input ever fails on it)
        P["ov_cap"] = OV_CAP0 if self.overlay else 0
        for j, kd in enumerate(kernels):
            for key, v in kd.items():
                if key == "ptype":
                    P["kernels"][j]["ptype"][:len(v)] = v
                else:
                    P["kernels"][j][key] = v
        P["max_ops"], P["mut_granule"], P["mut_redzone"] = mutation.max_ops, mutation.granule, mutation.redzone
        if mutation.max_ops > MAX_OPS:
            raise LoweringError(f"max_ops > {MAX_OPS}")
        P["window"], P["recent_weight"] = window, float(recent_weight)
        P["fanout"] = int(fanout)
        P["copy_src_mask"] = self.copy_src_mask
        P["term_phase"], P["jit_off"] = int(term_phase), int(not jit)
        P["master_seed"], P["keybase"], P["budget"] = master_seed & ((1 << 64) - 1), KEYBASE, budget
        P["diff_readback"], P["stop_first"] = int(diff_readback), int(stop_first)
        P["stop_class"] = -1 if stop_class is None else [c.value for c in CLASS_BY_CODE].index(stop_class)
        P["n_copyout_arg"] = len(copyout_args)
        for j, a in enumerate(copyout_args):
            P["copyout_arg"][j] = a
        P["readout_bytes_fixed"] = readout_fixed
        self.prog = P
        self.mutable = mutable

    def prog_bytes(self) -> bytes:
        return self.prog.tobytes()

    # ---- dedupe keys ---------------------------------------------------------------
    def key_parts(self, key: int):
        nl = len(self.labels) + 1
        site = key % nl
        rest = key // nl
        g = rest % (self.total_ins + 1)
        cls = rest // (self.total_ins + 1)
        if g == self.total_ins:
            kernel, iid = HOST, -1
        else:
            kernel, iid = self._kernel_of(g)
        label = "unmapped" if site == len(self.labels) else self.labels[site]
        return CLASS_BY_CODE[cls], kernel, iid, label

    def _kernel_of(self, g: int):
        for kidx, name in enumerate(self.kernel_names):
            kd = self.prog["kernels"][kidx]
            if kd["ins_base"] <= g < kd["ins_base"] + kd["n_ins"]:
                return name, g - int(kd["ins_base"])
        raise ValueError(g)


# ---- value / op codecs ------------------------------------------------------------------


def pack_values(tc: TestCase, specs):
    """TestCase -> (sfg_val[n_args] with data_off relative to the returned payload, payload)."""
    vals = np.zeros(len(specs), VAL)
    payload = bytearray()
    for j, v in enumerate(tc.args):
        if isinstance(v, IntValue):
            vals[j]["kind"], vals[j]["bits"] = V_I32, v.value & 0xFFFFFFFF
        elif isinstance(v, FloatValue):
            vals[j]["kind"], vals[j]["bits"] = V_F32, v.bits
        else:
            if len(v.extents) > 4:
                raise LoweringError("arrays with more than 4 extents are not lowered")
            vals[j]["kind"] = V_ARR
            vals[j]["elem"] = 1 if v.elem == "f32" else 0
            vals[j]["space"] = SPACE_INDEX[v.space]
            vals[j]["ndim"] = len(v.extents)
            vals[j]["ext"][:len(v.extents)] = v.extents
            vals[j]["count"] = v.count
            vals[j]["nbytes"] = len(v.data)
            if not -(1 << 40) < v.base_offset < (1 << 40):
                # the specialized kernels keep pointer registers in 64 bits when the
                # pointer parameters (base + base_offset) stay below 2^40 (jit.cu narrow_ok);
                # mutation keeps offsets within 2 * max(len, 4) (mutation.py:338-347)
                raise LoweringError(f"array base_offset {v.base_offset} outside +-2^40 is not lowered")
            vals[j]["base_offset"] = v.base_offset
            vals[j]["size_override"] = NO_OVERRIDE if v.size_override is None else v.size_override
            vals[j]["data_off"] = len(payload)
            payload += v.data + bytes((-len(v.data)) % 16)
    return vals, bytes(payload)


def unpack_values(vals, data: bytes, base: int = 0):
    """sfg_val row + payload bytes (data_off relative to ``base``) -> typed arg tuple."""
    out = []
    for v in vals:
        k = int(v["kind"])
        if k == V_I32:
            out.append(IntValue(struct.unpack("<i", struct.pack("<I", int(v["bits"])))[0]))
        elif k == V_F32:
            out.append(FloatValue(int(v["bits"])))
        else:
            off = int(v["data_off"]) - base
            nb = int(v["nbytes"])
            ov = int(v["size_override"])
            ext = tuple(int(e) for e in v["ext"][:int(v["ndim"])])
            out.append(ArrayValue(bytes(data[off:off + nb]), "f32" if v["elem"] == 1 else "i32", ext,
                                  SPACE_ORDER[int(v["space"])], int(v["base_offset"]),
                                  None if ov == NO_OVERRIDE else ov))
    return tuple(out)


_SPACES = [s.value for s in SPACE_ORDER]


def decode_op(o) -> MutationOp:
    """sfg_op -> MutationOp with the reference's exact parameter text (mutation.py:211-212)."""
    kind = M_KINDS[int(o["kind"])]
    arg = int(o["arg"])
    sub, byte, mask = int(o["sub"]), int(o["byte"]), int(o["mask"])
    if kind == "int_boundary":
        return MutationOp.make(kind, arg, which=("zero", "max", "min")[sub])
    if kind == "int_byte":
        if sub == 0:
            return MutationOp.make(kind, arg, mode="flip", byte=byte, mask=mask)
        return MutationOp.make(kind, arg, mode="add", delta=int(o["delta"]))
    if kind == "float_sign" or kind == "array_empty":
        return MutationOp.make(kind, arg)
    if kind == "float_exponent":
        if sub == 2:
            return MutationOp.make(kind, arg, pattern="bit", bit=byte)
        return MutationOp.make(kind, arg, pattern=("ones", "zeros")[sub])
    if kind == "float_mantissa":
        return MutationOp.make(kind, arg, mask=hex(mask))
    if kind == "float_byte":
        return MutationOp.make(kind, arg, byte=byte, mask=mask)
    if kind == "float_arith":
        return MutationOp.make(kind, arg, delta_bits=hex(mask))
    if kind == "array_extreme":
        return MutationOp.make(kind, arg, pattern=("zero", "max", "min")[sub])
    if kind == "array_dim":
        ext = str(mask) if sub == 1 else f"{mask}x{int(o['imask'])}"
        return MutationOp.make(kind, arg, extents=ext)
    if kind == "ptr_space":
        return MutationOp.make(kind, arg, target=_SPACES[sub])
    if kind == "ptr_offset":
        return MutationOp.make(kind, arg, delta=int(o["delta"]))
    inner = M_KINDS[int(o["inner"])]
    isub, ib, im = int(o["isub"]), int(o["ibyte"]), int(o["imask"])
    params = {"index": int(o["index"]), "inner": inner}
    if inner == "int_byte":
        params.update({"inner_mode": "flip", "inner_byte": ib, "inner_mask": im} if isub == 0
                      else {"inner_mode": "add", "inner_delta": int(o["delta"])})
    elif inner == "float_exponent":
        params.update({"inner_pattern": "bit", "inner_bit": ib} if isub == 2
                      else {"inner_pattern": ("ones", "zeros")[isub]})
    elif inner == "float_mantissa":
        params["inner_mask"] = hex(im)
    elif inner == "float_byte":
        params.update({"inner_byte": ib, "inner_mask": im})
    return MutationOp.make(kind, arg, **params)


def decode_verdict(v, low: Lowered, iteration: int, id_base: int) -> BugReport:
    """sfg_verdict (status FINDING) -> BugReport; ``id_base`` = campaign id of this
    input's first own allocation."""
    def aid(enc: int):
        if enc == 0:
            return None
        return enc if enc > 0 else id_base + (-enc - 1)

    kernel = HOST if int(v["kernel"]) < 0 else low.kernel_names[int(v["kernel"])]
    addr = (int(v["addr_hi"]) << 64) | (int(v["addr_lo"]) & ((1 << 64) - 1))
    label = int(v["label"])
    alloc = aid(int(v["alloc"]))
    space = int(v["space"])
    state = int(v["alloc_state"])
    return BugReport(CLASS_BY_CODE[int(v["bug_class"])], kernel, int(v["iid"]), int(v["ctaid"]), int(v["tid"]),
                     addr, int(v["width"]), bool(v["is_store"]), None if space == 255 else SPACE_ORDER[space],
                     MECHANISMS[int(v["mech"])], None if int(v["shadow"]) < 0 else int(v["shadow"]),
                     aid(int(v["prov"])), alloc, low.labels[label] if (label >= 0 and alloc is not None) else "",
                     int(v["alloc_base"]) if alloc is not None else 0,
                     int(v["alloc_size"]) if alloc is not None else 0,
                     ("LIVE", "FREED")[state] if (alloc is not None and state < 2) else "", iteration)


# ---- context-sensitive hashed coverage map (csrc/ctxmap.cu) ----

CTX_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def fmix64(k: int) -> int:
    k &= _M64
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & _M64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & _M64
    return k ^ (k >> 33)


def hit_bucket(c: int) -> int:
    """AFL hit-count class: 1, 2, 3, 4-7, 8-15, 16-31, 32-127, 128+ -> 1..8."""
    if c <= 3:
        return c
    for b, hi in ((4, 8), (5, 16), (6, 32), (7, 128)):
        if c < hi:
            return b
    return 8


def ctx_edge_hashes(low: "Lowered", manifest) -> np.ndarray:
    """Per dense edge: hash of (calling context, kernel, src, dst).  The calling
    context of a kernel is the launch chain of the COMPUTE phase up to its first
    launch (SIR has no call instruction)."""
    import hashlib
    chain = [op.kernel for op in manifest.phases[COMPUTE] if op.kind == "launch"]
    out = np.zeros(max(len(low.edge_names), 1), np.uint64)
    for e, (name, (a, b)) in enumerate(low.edge_names):
        ctx = chain[:chain.index(name) + 1] if name in chain else [name]
        h = 0x6A09E667F3BCC908
        for k in ctx:
            h = fmix64(h ^ int.from_bytes(hashlib.sha256(k.encode()).digest()[:8], "little"))
        out[e] = fmix64(h ^ (((a & 0xFFFFFFFF) << 32) | (b & 0xFFFFFFFF)))
    return out


def ctx_slot(edge_hash: int, count: int, bits: int) -> int:
    return fmix64(int(edge_hash) ^ ((hit_bucket(count) * CTX_GOLDEN) & _M64)) & ((1 << bits) - 1)
