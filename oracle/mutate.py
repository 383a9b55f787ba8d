"""ORACLE (test infrastructure): type-aware mutation, restated.

Follows ``simt_forge/mutation.py``:
  operators  mutate_int :258-278, _float_bits_op :281-306, _int_bits_op :313-315,
             mutate_array :318-357, apply_op :360-365
  generators MutationSchedule.next_int_op :371-386, _gen_int_byte :396-401,
             _gen_float_op :404-422, _offset_palette :425-438,
             _gen_array_op :441-474, _gen_extents :477-487, generate_op :490-496
  driver     mutate_testcase :499-518 (split into draw_picks + finish_child so the
             batched-round driver can prefix-sum the boundary rotation counts)
Data types come from the product's host data model (plain records).
"""

from __future__ import annotations

import struct
from dataclasses import replace

from paper_2603_05725_b200.sir import SPACE_ORDER, MemSpace
from paper_2603_05725_b200.testcase import (F32_MAX_BITS, F32_MIN_BITS, I32_MAX, I32_MIN,
                                            ArrayValue, FloatValue, IntValue, MutationError,
                                            MutationOp, TestCase, bits_f32, f32_bits)

TYPE_AWARE_WEIGHT = 0.4
BOUNDARY = ("zero", "max", "min")
ARITH_DELTAS = (1.0, -1.0, 0.5, 2.0, 1024.0, 0.001)
INT_DELTAS = (-16, -4, -2, -1, 1, 2, 4, 16)


def _f32_add_bits(a_bits: int, b_bits: int) -> int:
    # double add of two binary32 values, narrowed once (x86 NaN rules via ctypes)
    return f32_bits(bits_f32(a_bits) + bits_f32(b_bits))


def float_bits_op(bits: int, op: MutationOp) -> int:
    k = op.kind
    if k == "float_sign":
        return bits ^ 0x80000000
    if k == "float_exponent":
        pat = op.param("pattern")
        if pat == "ones":
            return bits | 0x7F800000
        if pat == "zeros":
            return bits & 0x807FFFFF
        if pat == "bit":
            return bits ^ (1 << (23 + int(op.param("bit"))))
        raise MutationError(f"bad exponent pattern {pat!r}")
    if k == "float_mantissa":
        mask = int(op.param("mask"), 0) & 0x007FFFFF
        if not mask:
            raise MutationError("float_mantissa needs a nonzero mask")
        return bits ^ mask
    if k == "float_byte":
        return bits ^ ((int(op.param("mask")) & 0xFF) << (8 * int(op.param("byte"))))
    if k == "float_arith":
        return _f32_add_bits(bits, int(op.param("delta_bits"), 0))
    raise MutationError(f"{k} does not apply to f32")


def int_op(v: int, op: MutationOp) -> int:
    if op.kind == "int_boundary":
        which = op.param("which")
        if which not in BOUNDARY:
            raise MutationError(f"bad boundary {which!r}")
        return {"zero": 0, "max": I32_MAX, "min": I32_MIN}[which]
    if op.kind == "int_byte":
        mode = op.param("mode")
        if mode == "flip":
            return IntValue(v ^ ((int(op.param("mask")) & 0xFF) << (8 * int(op.param("byte"))))).value
        if mode == "add":
            return IntValue(v + int(op.param("delta"))).value
        raise MutationError(f"bad int_byte mode {mode!r}")
    raise MutationError(f"{op.kind} does not apply to i32")


def array_op(v: ArrayValue, op: MutationOp) -> ArrayValue:
    k = op.kind
    if k == "array_extreme":
        pat = op.param("pattern")
        table = ({"zero": 0, "max": F32_MAX_BITS, "min": F32_MIN_BITS} if v.elem == "f32"
                 else {"zero": 0, "max": I32_MAX, "min": 1 << 31})
        return replace(v, data=struct.pack("<I", table[pat]) * v.count)
    if k == "array_dim":
        txt = op.param("extents")
        ext = (0,) if txt == "0" else tuple(int(t) for t in txt.split("x"))
        n = 1
        for e in ext:
            n *= e
        want = 4 * n
        data = v.data[:want] if want <= len(v.data) else v.data + bytes(want - len(v.data))
        return replace(v, data=data, extents=ext)
    if k == "array_empty":
        return replace(v, data=b"", extents=(0,))
    if k == "ptr_space":
        return replace(v, space=MemSpace(op.param("target")))
    if k == "ptr_offset":
        lim = 2 * max(len(v.data), 4)
        d = max(-lim, min(lim, int(op.param("delta"))))
        return replace(v, base_offset=v.base_offset + d)
    if k == "array_elem":
        idx = int(op.param("index"))
        if not 0 <= idx < v.count:
            raise MutationError(f"array_elem index {idx} out of range")
        inner = MutationOp(op.param("inner"), op.arg,
                           tuple((key[6:], val) for key, val in op.params if key.startswith("inner_")))
        bits = struct.unpack_from("<I", v.data, 4 * idx)[0]
        if v.elem == "f32":
            bits = float_bits_op(bits, inner)
        else:
            signed = bits - (1 << 32) if bits & 0x80000000 else bits
            bits = int_op(signed, inner) & 0xFFFFFFFF
        buf = bytearray(v.data)
        struct.pack_into("<I", buf, 4 * idx, bits & 0xFFFFFFFF)
        return replace(v, data=bytes(buf))
    raise MutationError(f"{k} does not apply to arrays")


def apply_op(value, op: MutationOp):
    if isinstance(value, IntValue):
        return IntValue(int_op(value.value, op))
    if isinstance(value, FloatValue):
        return FloatValue(float_bits_op(value.bits, op))
    return array_op(value, op)


def apply_trace(parent: TestCase, trace, rng_seed: int = 0) -> TestCase:
    args = list(parent.args)
    for op in trace:
        args[op.arg] = apply_op(args[op.arg], op)
    return TestCase(tuple(args), rng_seed, parent.id, tuple(trace))


# -- generation ----------------------------------------------------------------------


def gen_int_byte(arg: int, rng) -> MutationOp:
    if rng.random() < 0.5:
        return MutationOp.make("int_byte", arg, mode="flip", byte=rng.integers(0, 4),
                               mask=rng.integers(1, 256))
    return MutationOp.make("int_byte", arg, mode="add", delta=rng.choice(list(INT_DELTAS)))


def int_op_for_count(arg: int, count: int, rng) -> MutationOp:
    """``MutationSchedule.next_int_op`` given the arg's rotation count."""
    if count < 3:
        return MutationOp.make("int_boundary", arg, which=BOUNDARY[count])
    if rng.random() < TYPE_AWARE_WEIGHT:
        return MutationOp.make("int_boundary", arg, which=rng.choice(BOUNDARY))
    return gen_int_byte(arg, rng)


def gen_float_op(arg: int, rng) -> MutationOp:
    if rng.random() < TYPE_AWARE_WEIGHT:
        pick = rng.integers(0, 4)
        if pick == 0:
            return MutationOp.make("float_sign", arg)
        if pick == 1:
            pat = rng.choice(["ones", "zeros", "bit"])
            if pat == "bit":
                return MutationOp.make("float_exponent", arg, pattern="bit", bit=rng.integers(0, 8))
            return MutationOp.make("float_exponent", arg, pattern=pat)
        if pick == 2:
            return MutationOp.make("float_mantissa", arg, mask=hex(rng.integers(1, 1 << 23)))
        d = rng.choice(ARITH_DELTAS)
        return MutationOp.make("float_arith", arg, delta_bits=hex(f32_bits(d)))
    return MutationOp.make("float_byte", arg, byte=rng.integers(0, 4), mask=rng.integers(1, 256))


def offset_palette(size: int, granule: int = 4, redzone: int = 32):
    g, rz = granule, redzone
    size = max(size, g)
    mags = {g, 2 * g, rz, rz + g, 2 * rz, 2 * rz + g, 2 * rz - g, size, size + 2 * rz,
            size + rz, 2 * size}
    out = []
    for m in sorted(mags):
        if 0 < m <= 2 * size:
            out += [m, -m]
    return out or [g, -g]


def gen_extents(v: ArrayValue, rng) -> str:
    n = v.count
    if n >= 2:
        opts = [str(n // 2), f"{n}x2"] + ([f"2x{n // 2}"] if n % 2 == 0 else [])
    else:
        opts = [str(2 * n + 2)]
    return rng.choice(opts)


def gen_array_op(arg: int, v: ArrayValue, rng, granule=4, redzone=32) -> MutationOp:
    others = [s.value for s in SPACE_ORDER if s != v.space]
    if v.count == 0:
        pick = rng.integers(0, 3)
        if pick == 0:
            return MutationOp.make("array_dim", arg, extents="4")
        if pick == 1:
            return MutationOp.make("ptr_space", arg, target=rng.choice(others))
        return MutationOp.make("ptr_offset", arg,
                               delta=rng.choice(offset_palette(len(v.data), granule, redzone)))
    if rng.random() < TYPE_AWARE_WEIGHT:
        pick = rng.integers(0, 5)
        if pick == 0:
            return MutationOp.make("array_extreme", arg, pattern=rng.choice(["zero", "max", "min"]))
        if pick == 1:
            return MutationOp.make("array_dim", arg, extents=gen_extents(v, rng))
        if pick == 2:
            return MutationOp.make("array_empty", arg)
        if pick == 3:
            return MutationOp.make("ptr_space", arg, target=rng.choice(others))
        return MutationOp.make("ptr_offset", arg,
                               delta=rng.choice(offset_palette(len(v.data), granule, redzone)))
    index = rng.integers(0, v.count)
    if v.elem == "f32":
        inner = gen_float_op(arg, rng)
        while inner.kind == "float_arith":
            inner = gen_float_op(arg, rng)
    else:
        inner = gen_int_byte(arg, rng)
    params = {"index": index, "inner": inner.kind}
    params.update({f"inner_{k}": val for k, val in inner.params})
    return MutationOp.make("array_elem", arg, **params)


def draw_picks(specs, rng, max_ops: int = 3):
    """First half of ``mutate_testcase`` (:502-511): op count + distinct args."""
    mutable = [i for i, s in enumerate(specs) if not s.fixed]
    if not mutable:
        raise MutationError("no mutable arguments")
    cap = min(max_ops, len(mutable))
    n_ops = 1 + rng.geometric_small(0.5, cap - 1)
    pool = list(mutable)
    return [pool.pop(rng.integers(0, len(pool))) for _ in range(n_ops)]


def finish_child(parent: TestCase, picks, int_counts: dict, rng, granule=4, redzone=32) -> TestCase:
    """Second half (:512-518).  ``int_counts`` is updated in place (the rotation
    state of ``MutationSchedule``)."""
    args = list(parent.args)
    ops = []
    for a in picks:
        v = args[a]
        if isinstance(v, IntValue):
            c = int_counts.get(a, 0)
            int_counts[a] = c + 1
            op = int_op_for_count(a, c, rng)
        elif isinstance(v, FloatValue):
            op = gen_float_op(a, rng)
        else:
            op = gen_array_op(a, v, rng, granule, redzone)
        args[a] = apply_op(v, op)
        ops.append(op)
    return TestCase(tuple(args), rng.u64(), parent.id, tuple(ops))


def mutate_testcase(parent: TestCase, specs, int_counts: dict, rng, max_ops=3,
                    granule=4, redzone=32) -> TestCase:
    return finish_child(parent, draw_picks(specs, rng, max_ops), int_counts, rng, granule, redzone)
