"""ORACLE (test infrastructure): sequential SIMT interpreter, restated.

Follows ``simt_forge/executor.py``: f32/i32/cvt helpers :42-65, arg binding
:167-188, per-instruction semantics ``_exec_one`` :210-377 and the block-major,
thread-major, run-to-completion ``launch`` loop with first-bug-stop and the
per-thread retired-instruction budget :390-424.  f32 arithmetic is host double
math narrowed through ``ctypes.c_float`` exactly like the reference, so NaN
payloads follow the x86-64 host rules the reference exhibits.
"""

from __future__ import annotations

import ctypes
import math
import struct

from paper_2603_05725_b200.sir import Opcode, ScalarType

from .memory import check_access

_F = struct.Struct("<f")
_I = struct.Struct("<i")
_Q = struct.Struct("<Q")
_H = struct.Struct("<H")


def f32(x: float) -> float:
    return ctypes.c_float(x).value


def wrap32(v: int) -> int:
    return ((v + (1 << 31)) & 0xFFFFFFFF) - (1 << 31)


def cvt_to_i32(v: float) -> int:
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


class Outcome:
    __slots__ = ("status", "report", "retired", "threads_completed")

    def __init__(self, status, report, retired, done):
        self.status, self.report, self.retired, self.threads_completed = status, report, retired, done


def launch(program, img, kname, grid, block, args, *, coverage=None, budget=1_000_000,
           iteration=-1):
    """``args``: list of (ScalarType, value, prov).  Returns Outcome with status
    'COMPLETED' | 'SANITIZER_STOP' | 'BUDGET_EXHAUSTED'."""
    k = program.kernels[kname]
    pre_r, pre_f, pre_a, pre_p = [], [], [], []
    for p, (ty, val, prov) in zip(k.params, args):
        if p.type == ScalarType.I32:
            pre_r.append(wrap32(int(val)))
        elif p.type == ScalarType.F32:
            pre_f.append(f32(float(val)))
        else:
            pre_a.append(int(val))
            pre_p.append(prov)
    if coverage is not None:
        coverage.record_launch(kname)
    ins_list = k.instructions
    n = k.register_count
    total = 0
    done = 0
    for ctaid in range(grid):
        for tid in range(block):
            r = pre_r + [0] * (n - len(pre_r))
            f = pre_f + [0.0] * (n - len(pre_f))
            a = pre_a + [0] * (n - len(pre_a))
            ap = pre_p + [None] * (n - len(pre_p))
            pr = [False] * n
            pc = 0
            retired = 0
            while True:
                ins = ins_list[pc]
                op = ins.opcode
                retired += 1
                if op == Opcode.EXIT:
                    total += retired
                    done += 1
                    break
                if op == Opcode.BRA:
                    taken = True if ins.pred is None else (pr[ins.pred[1]] != ins.pred_negate)
                    npc = ins.target_iid if taken else pc + 1
                    if coverage is not None:
                        coverage.record_edge(kname, ins.block, ins_list[npc].block)
                    pc = npc
                    if retired >= budget:
                        return Outcome("BUDGET_EXHAUSTED", None, total + retired, done)
                    continue
                if op == Opcode.LD or op == Opcode.ST:
                    base, off = ins.addr
                    addr = a[base[1]] + off
                    st = op == Opcode.ST
                    rep = check_access(img, addr, ins.width, ins.space, ap[base[1]], kernel=kname,
                                       iid=ins.iid, ctaid=ctaid, tid=tid, is_store=st,
                                       iteration=iteration)
                    if rep is not None:
                        return Outcome("SANITIZER_STOP", rep, total + retired, done)
                    kind = ins.mem_kind
                    if st:
                        s = ins.srcs[0]
                        reg = isinstance(s, tuple)
                        if kind == "f32":
                            raw = _F.pack(f[s[1]] if reg else f32(float(s)))
                        elif kind == "b32":
                            raw = _I.pack(r[s[1]] if reg else wrap32(int(s)))
                        elif kind == "b64":
                            raw = _Q.pack(a[s[1]] & 0xFFFFFFFFFFFFFFFF)
                        elif kind == "b16":
                            raw = _H.pack((r[s[1]] if reg else int(s)) & 0xFFFF)
                        else:
                            raw = bytes([(r[s[1]] if reg else int(s)) & 0xFF])
                        img.write(addr, raw)
                    else:
                        raw = img.read(addr, ins.width)
                        d = ins.dst[1]
                        if kind == "f32":
                            f[d] = _F.unpack(raw)[0]
                        elif kind == "b32":
                            r[d] = _I.unpack(raw)[0]
                        elif kind == "b64":
                            a[d] = _Q.unpack(raw)[0]
                            ap[d] = None
                        elif kind == "b16":
                            r[d] = _H.unpack(raw)[0]
                        else:
                            r[d] = raw[0]
                elif op == Opcode.MOV:
                    c, d = ins.dst
                    s = ins.srcs[0]
                    reg = isinstance(s, tuple)
                    if c == "r":
                        r[d] = r[s[1]] if reg else wrap32(int(s))
                    elif c == "f":
                        f[d] = f[s[1]] if reg else f32(float(s))
                    elif c == "a":
                        a[d], ap[d] = (a[s[1]], ap[s[1]]) if reg else (int(s), None)
                    else:
                        pr[d] = pr[s[1]]
                elif op in (Opcode.ADD, Opcode.SUB, Opcode.MUL):
                    c, d = ins.dst
                    s1, s2 = ins.srcs
                    if c == "a":
                        delta = r[s2[1]] if isinstance(s2, tuple) else int(s2)
                        a[d] = a[s1[1]] + delta if op == Opcode.ADD else a[s1[1]] - delta
                        ap[d] = ap[s1[1]]
                    else:
                        x = r[s1[1]] if isinstance(s1, tuple) else int(s1)
                        y = r[s2[1]] if isinstance(s2, tuple) else int(s2)
                        r[d] = wrap32(x + y if op == Opcode.ADD else x - y if op == Opcode.SUB else x * y)
                elif op in (Opcode.FADD, Opcode.FSUB, Opcode.FMUL):
                    s1, s2 = ins.srcs
                    x = f[s1[1]] if isinstance(s1, tuple) else f32(float(s1))
                    y = f[s2[1]] if isinstance(s2, tuple) else f32(float(s2))
                    f[ins.dst[1]] = f32(x + y if op == Opcode.FADD else x - y if op == Opcode.FSUB else x * y)
                elif op == Opcode.SETP:
                    s1, s2 = ins.srcs
                    fl = any((isinstance(s, tuple) and s[0] == "f") or isinstance(s, float) for s in (s1, s2))
                    if fl:
                        x = f[s1[1]] if isinstance(s1, tuple) else f32(float(s1))
                        y = f[s2[1]] if isinstance(s2, tuple) else f32(float(s2))
                    else:
                        x = r[s1[1]] if isinstance(s1, tuple) else int(s1)
                        y = r[s2[1]] if isinstance(s2, tuple) else int(s2)
                    cm = ins.cmp
                    pr[ins.dst[1]] = (x == y if cm == "eq" else x != y if cm == "ne" else x < y if cm == "lt"
                                      else x <= y if cm == "le" else x > y if cm == "gt" else x >= y)
                elif op == Opcode.CVT:
                    s = ins.srcs[0]
                    if ins.cvt[0] == ScalarType.F32:
                        f[ins.dst[1]] = f32(float(r[s[1]] if isinstance(s, tuple) else int(s)))
                    else:
                        r[ins.dst[1]] = cvt_to_i32(f[s[1]] if isinstance(s, tuple) else float(s))
                elif op == Opcode.SREG:
                    r[ins.dst[1]] = {"tid": tid, "ntid": block, "ctaid": ctaid, "nctaid": grid}[ins.sreg]
                nb = ins_list[pc + 1].block
                if nb != ins.block and coverage is not None:
                    coverage.record_edge(kname, ins.block, nb)
                pc += 1
                if retired >= budget:
                    return Outcome("BUDGET_EXHAUSTED", None, total + retired, done)
    return Outcome("COMPLETED", None, total, done)
