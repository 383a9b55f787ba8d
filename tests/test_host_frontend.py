"""CPU tests: host front end digests, lowering of every bundled harness, the
C-ABI library's exports and record layouts (no GPU needed)."""

import ctypes
import re

import pytest

from conftest import bench_manifest, bench_names, golden
from paper_2603_05725_b200 import _native
from paper_2603_05725_b200 import lowering as lw
from paper_2603_05725_b200.baseline import MemConfig, build_baseline, record_table
from paper_2603_05725_b200.engine import MutationConfig
from paper_2603_05725_b200.testcase import argspec_digest

VARIANTS = ("spatial_oob", "temporal_uaf", "space_mismatch", "provenance_escape")


@pytest.mark.parametrize("key", sorted(golden("ref_fuzzloop.json")))
def test_digests_match_reference(key):
    name = key.split("/")[0]
    m = bench_manifest(name)
    summ = golden("ref_fuzzloop.json")[key]["summary"]
    prog, man, arg = re.search(r"program=(\w+) manifest=(\w+) argspec=(\w+)", summ).groups()
    assert m.program_digest == prog
    assert m.digest == man
    assert argspec_digest(m.argspecs) == arg


@pytest.mark.parametrize("name", bench_names())
def test_every_harness_lowers(name):
    for variant in (None,) + VARIANTS:
        m = bench_manifest(name, variant)
        base = build_baseline(m, m.seed(11), MemConfig())
        low = lw.Lowered(m, base, mem=MemConfig(), mutation=MutationConfig(), master_seed=11, budget=10**6,
                         window=256, recent_weight=4.0)
        recs = record_table(base, low.labels)
        assert len(low.ins) == sum(len(k.instructions) for k in m.program.kernels.values())
        assert low.n_edges == sum(len(k.edges) for k in m.program.kernels.values())
        assert len(recs) >= 2
        # INIT lays out ws then lut exactly like the reference allocator
        assert base.named["ws"][0] == 0x10000020
        assert base.named["lut"][0] == 0x10800060
        for key in range(0, low.n_keys, max(1, low.n_keys // 50)):
            low.key_parts(key)


def test_library_exports_and_layouts():
    lib = _native.lib()
    import re
    declared = set(re.findall(r"\b(sfg_[a-z0-9_]+)\s*\(", _native.HEADER.read_text()))
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert lib.sfg_abi_version() == 5
    sizes = [lib.sfg_layout_probe(i) for i in range(14)]
    want = [lw.INS.itemsize, lw.KERNEL.itemsize, lw.HOSTOP.itemsize, lw.BINDING.itemsize, lw.REC.itemsize,
            lw.VAL.itemsize, lw.OP.itemsize, lw.CHILD.itemsize, lw.ENTRY.itemsize, lw.VERDICT.itemsize,
            lw.PROG.itemsize, lw.PROG.fields["kernels"][1], lw.PROG.fields["recent_weight"][1],
            lw.PROG.fields["copyout_arg"][1]]
    assert sizes == want


def test_header_declares_every_export():
    text = (_native.HEADER).read_text()
    for sym in _native.EXPORTS:
        assert re.search(rf"\b{sym}\s*\(", text), sym


def test_op_codec_roundtrip_against_oracle_text():
    """decode_op reproduces MutationOp.encode() text for ops the oracle generates."""
    import numpy as np
    from oracle.loop import batched_loop
    m = bench_manifest("rotm")
    res = batched_loop(m, master_seed=5, iterations=300, round_size=100)
    seen = 0
    for r in res.records[1:]:
        for op in r["child"].trace:
            o = np.zeros(1, lw.OP)[0]
            _encode_for_test(o, op)
            assert lw.decode_op(o).encode() == op.encode()
            seen += 1
    assert seen > 300


def _encode_for_test(o, op):
    """Test-side encoder (device ops are produced by the kernel; this mirrors the layout)."""
    kind = lw.M_INDEX[op.kind]
    o["kind"], o["arg"] = kind, op.arg
    p = dict(op.params)
    sub = {"zero": 0, "max": 1, "min": 2, "ones": 0, "zeros": 1, "bit": 2, "flip": 0, "add": 1,
           "global": 0, "shared": 1, "local": 2}
    if op.kind in ("int_boundary",):
        o["sub"] = sub[p["which"]]
    elif op.kind == "int_byte":
        o["sub"] = sub[p["mode"]]
        if p["mode"] == "flip":
            o["byte"], o["mask"] = int(p["byte"]), int(p["mask"])
        else:
            o["delta"] = int(p["delta"])
    elif op.kind == "float_exponent":
        o["sub"] = sub[p["pattern"]]
        if p["pattern"] == "bit":
            o["byte"] = int(p["bit"])
    elif op.kind in ("float_mantissa",):
        o["mask"] = int(p["mask"], 0)
    elif op.kind == "float_byte":
        o["byte"], o["mask"] = int(p["byte"]), int(p["mask"])
    elif op.kind == "float_arith":
        o["mask"] = int(p["delta_bits"], 0)
    elif op.kind == "array_extreme":
        o["sub"] = sub[p["pattern"]]
    elif op.kind == "array_dim":
        e = [int(x) for x in p["extents"].split("x")]
        o["sub"], o["mask"] = len(e), e[0]
        if len(e) == 2:
            o["imask"] = e[1]
    elif op.kind == "ptr_space":
        o["sub"] = sub[p["target"]]
    elif op.kind == "ptr_offset":
        o["delta"] = int(p["delta"])
    elif op.kind == "array_elem":
        o["index"] = int(p["index"])
        inner = p["inner"]
        o["inner"] = lw.M_INDEX[inner]
        if inner == "int_byte":
            o["isub"] = sub[p["inner_mode"]]
            if p["inner_mode"] == "flip":
                o["ibyte"], o["imask"] = int(p["inner_byte"]), int(p["inner_mask"])
            else:
                o["delta"] = int(p["inner_delta"])
        elif inner == "float_exponent":
            o["isub"] = sub[p["inner_pattern"]]
            if p["inner_pattern"] == "bit":
                o["ibyte"] = int(p["inner_bit"])
        elif inner == "float_mantissa":
            o["imask"] = int(p["inner_mask"], 0)
        elif inner == "float_byte":
            o["ibyte"], o["imask"] = int(p["inner_byte"]), int(p["inner_mask"])


@pytest.mark.parametrize("name", ["dot", "amax", "vadd", "ctxchain"])  # the GPU suite compiles every harness
def test_jit_source_compiles_for_sm100a(name):
    """The specialized execute kernel (SIR -> CUDA C++) NVRTC-compiles for sm_100a."""
    import sys
    sys.path.insert(0, str(_native.PKG.parent / "tools"))
    from jit_check import check
    if name in ("matmul", "vadd", "ctxchain"):
        from paper_2603_05725_b200.workloads import load
        m = load(name)
    else:
        m = bench_manifest(name)
    rc, cubin_bytes, text = check(m)
    assert rc == 0, text[:2000]
    assert cubin_bytes > 0
    assert "sfg_jit_execute" in text


def test_sample_valid_testcase_matches_reference_seeds():
    """Seed corpora for C4: sample_valid_testcase draw for draw as the reference
    (golden seeds generated by the reference's own function)."""
    from conftest import golden, workload_manifest
    from paper_2603_05725_b200.testcase import Stream, sample_valid_testcase, serialize_testcase
    m = workload_manifest("structcfg")
    want = golden("ref_workloads.json")["structcfg"]["seeds"]
    for k, text in enumerate(want):
        assert serialize_testcase(sample_valid_testcase(m.argspecs, Stream(11, (7 << 40) + k))) == text


def _control_args(m):
    import ctypes
    from paper_2603_05725_b200.baseline import MemConfig, build_baseline
    from paper_2603_05725_b200.engine import MutationConfig
    from paper_2603_05725_b200.lowering import Lowered
    base = build_baseline(m, m.seed(11), MemConfig())
    low = Lowered(m, base, mem=MemConfig(), mutation=MutationConfig(), master_seed=11, budget=10**6, window=256,
                  recent_weight=4.0)
    P = low.prog_bytes()
    L = _native.lib()
    mask = L.sfg_control_mask(P, len(P), low.ins.ctypes.data, low.hostops.ctypes.data, len(low.hostops),
                              low.binds.ctypes.data)
    return {s.name for a, s in enumerate(m.argspecs) if mask >> a & 1}


def test_control_taint_mask():
    """sfg_order's signature covers the arguments that can steer control: those
    reaching a setp (loop bounds, compared values) and those reaching a load or
    store address (the sanitizer's verdict stops the thread), not pure data such
    as float scale factors (csrc/abi.cu control_arg_mask)."""
    from paper_2603_05725_b200.workloads import load
    assert _control_args(load("matmul")) == {"a", "b", "c", "m", "n", "k", "lda", "ldb", "ldc"}
    assert _control_args(load("vadd")) == {"x", "y", "z", "n"}
    assert _control_args(load("structcfg")) == {"cfg", "x", "y"}      # not the f32 alpha
    # amax compares loaded elements: the array steers control through its contents
    amax = _control_args(bench_manifest("amax"))
    assert "n" in amax and "x" in amax
    assert _control_args(bench_manifest("copy")) == {"x", "y", "n"}
    assert _control_args(bench_manifest("rotm")) == {"x", "y", "flag", "n"}   # not h11..h22
    assert _control_args(bench_manifest("axpy")) == {"x", "y", "n"}          # not the scale a


def test_bench_reference_arm_cpu():
    """bench.py --impl reference: the unmodified reference fuzz_loop from
    baseline/_ref when it is installed, else the CPU port of the reference loop, on
    the bench workload in clock-bounded windows; one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--ref-seconds", "1"], cwd=root, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "execs/s"
    want = "reference" if (root / "baseline" / "_ref" / "simt_forge").is_dir() else "port"
    assert line["cpu_baseline"]["kind"] == want and line["cpu_baseline"]["cores"] >= 1
    # the port measures clock windows; the reference arm's step also holds the
    # campaign processes' start-up (numpy import, manifest load, INIT)
    hi = 1500 if want == "port" else 30000
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and 900 <= line["ms_per_step"] <= hi


def test_jit_pointer_register_width():
    """The specializer keeps simulated pointer registers in int64 only when the
    kernel cannot push them past 2^62 (pointer params, small immediates, i32
    offsets, budget < 2^30): matmul is narrow; a 64-bit load into a pointer
    register or a near-2^63 immediate keeps the 128-bit form (csrc/jit.cu narrow_ok)."""
    import ctypes
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import jit_check
    from paper_2603_05725_b200.manifest import harness_from_text
    from paper_2603_05725_b200.workloads import load
    from test_gpu_parity import WIDE_MAN, WIDE_SIR
    rc, _, src = jit_check.check(load("matmul"))
    assert rc == 0 and "int64_t a0 =" in src and "i128 a0 =" not in src
    rc, _, src = jit_check.check(harness_from_text(WIDE_MAN, WIDE_SIR, "widereg/harness.man"))
    assert rc == 0 and "i128 a1 =" in src


def test_jit_load_quieting_only_when_observable():
    """A loaded f32 is quieted (the reference loads through a double) only when
    its register's bits can be observed -- copied by a mov or stored; operands
    of fadd/fmul/setp/cvt cannot tell a signaling NaN from its quieted form
    (csrc/jit.cu f_observers).  matmul feeds its loads to fmul only; copy
    stores what it loads."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import jit_check
    from paper_2603_05725_b200.workloads import load
    rc, _, src = jit_check.check(load("matmul"))
    assert rc == 0 and "sfg_quiet((uint32_t)v_)" not in src and "= (uint32_t)v_;" in src
    rc, _, src = jit_check.check(bench_manifest("copy"))
    assert rc == 0 and "sfg_quiet((uint32_t)v_)" in src
