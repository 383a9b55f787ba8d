"""Capacity limits of the device tables are load-time LoweringErrors, never a
mid-campaign failure.  Each harness below is valid for the
reference (which has no such tables); the device path refuses it before any
device work, with the limit in the message.  Copy-on-write overlay size, edge
counters and the TERM / INIT / copy_in features are not limits (see
tests/test_phase_features.py)."""

import pytest

from paper_2603_05725_b200.baseline import MemConfig, build_baseline
from paper_2603_05725_b200.engine import MutationConfig
from paper_2603_05725_b200.lowering import LoweringError, Lowered, pack_values
from paper_2603_05725_b200.manifest import harness_from_text


def lower(man, sir, *, mutation=None):
    m = harness_from_text(man, sir, "limits/harness.man")
    base = build_baseline(m, m.seed(1), MemConfig())
    return m, Lowered(m, base, mem=MemConfig(), mutation=mutation or MutationConfig(), master_seed=1,
                      budget=10 ** 6, window=256, recent_weight=4.0)


def test_limits_accept_the_bundled_shape():
    sir = "kernel k(x:ptr.global, n:i32) regs=64\n  st.global.b32 [%a0], %r0\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=4 extents=2x2 seed=zeros lo=0 hi=9\n"
           "argspec n i32 seed=1 lo=0 hi=9\n\ncompute:\n  launch k grid=1 block=1 args=arg:0,arg:1\n")
    _, low = lower(man, sir)          # 64 registers (was 32) are lowered
    assert low.n_edges == 0


def test_register_count_limit():
    sir = "kernel k(x:ptr.global) regs=65\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=4 seed=zeros lo=0 hi=9\n\n"
           "compute:\n  launch k grid=1 block=1 args=arg:0\n")
    with pytest.raises(LoweringError, match="regs=65 exceeds 64"):
        lower(man, sir)


def test_static_edge_limit():
    body = "".join(f"  setp.eq %p0, %r0, {i}\n  bra %p0, fin\n  add %r1, %r1, 1\n" for i in range(520))
    sir = "kernel k(x:ptr.global, n:i32) regs=4\n" + body + "fin:\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=4 seed=zeros lo=0 hi=9\n"
           "argspec n i32 seed=1 lo=0 hi=9\n\ncompute:\n  launch k grid=1 block=1 args=arg:0,arg:1\n")
    with pytest.raises(LoweringError, match="static edges exceed 1024"):
        lower(man, sir)


def test_argspec_limit():
    specs = "".join(f"argspec n{i} i32 seed=1 lo=0 hi=9\n" for i in range(17))
    params = ", ".join(f"n{i}:i32" for i in range(17))
    sir = f"kernel k({params}) regs=20\n  exit\n"
    man = ("program k.sir\n\n" + specs + "\ncompute:\n  launch k grid=1 block=1 args=" +
           ",".join(f"arg:{i}" for i in range(17)) + "\n")
    with pytest.raises(LoweringError, match="more than 16"):
        lower(man, sir)


def test_max_ops_limit():
    sir = "kernel k(x:ptr.global) regs=4\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=4 seed=zeros lo=0 hi=9\n\n"
           "compute:\n  launch k grid=1 block=1 args=arg:0\n")
    with pytest.raises(LoweringError, match="max_ops > 3"):
        lower(man, sir, mutation=MutationConfig(max_ops=4))


def test_per_input_allocation_table_limit():
    allocs = "".join(f"  alloc b{i} global 64\n" for i in range(30))
    specs = "".join(f"argspec x{i} ptr global i32 count=4 seed=zeros lo=0 hi=9\n" for i in range(11))
    sir = "kernel k(" + ", ".join(f"x{i}:ptr.global" for i in range(11)) + ") regs=12\n  exit\n"
    frees = "".join(f"  free b{i}\n" for i in range(30))
    man = ("program k.sir\n\n" + specs + "\ninit:\n" + allocs + "compute:\n  launch k grid=1 block=1 args=" +
           ",".join(f"arg:{i}" for i in range(11)) + "\nterm:\n" + frees)
    with pytest.raises(LoweringError, match="per-input table"):
        lower(man, sir)


def test_quarantine_limit():
    init = "".join(f"  alloc i{i} global 64\n  free i{i}\n" for i in range(19))      # 19 quarantined
    comp = "".join(f"  alloc c{i} global 64\n  free c{i}\n" for i in range(13)) + "  free i0\n"
    term = "".join(f"  free i{i}\n" for i in range(19))
    sir = "kernel k(x:ptr.global) regs=4\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=4 seed=zeros lo=0 hi=9\n\n"
           "init:\n" + init + "compute:\n  launch k grid=1 block=1 args=arg:0\n" + comp + "term:\n" + term)
    with pytest.raises(LoweringError, match="quarantine"):
        lower(man, sir)


def test_extents_and_base_offset_limits():
    from paper_2603_05725_b200.testcase import ArrayValue, TestCase
    from paper_2603_05725_b200.sir import MemSpace
    sir = "kernel k(x:ptr.global) regs=4\n  exit\n"
    man = ("program k.sir\n\nargspec x ptr global i32 count=32 extents=2x2x2x2x2 seed=zeros lo=0 hi=9\n\n"
           "compute:\n  launch k grid=1 block=1 args=arg:0\n")
    m = harness_from_text(man, sir, "limits/harness.man")
    with pytest.raises(LoweringError, match="more than 4 extents"):
        pack_values(m.seed(1), m.argspecs)
    far = TestCase((ArrayValue(bytes(16), "i32", (4,), MemSpace.GLOBAL, base_offset=1 << 41),), 0)
    with pytest.raises(LoweringError, match="base_offset"):
        pack_values(far, m.argspecs)
