"""Generate + NVRTC-compile the specialized execute kernel for a harness (CPU only)."""
import ctypes, json, sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_2603_05725_b200 import _native
from paper_2603_05725_b200.baseline import MemConfig, build_baseline
from paper_2603_05725_b200.engine import MutationConfig
from paper_2603_05725_b200.lowering import Lowered
from paper_2603_05725_b200.manifest import harness_from_text


def check(m, dump=None):
    base = build_baseline(m, m.seed(11), MemConfig())
    low = Lowered(m, base, mem=MemConfig(), mutation=MutationConfig(), master_seed=11, budget=10**6, window=256,
                  recent_weight=4.0)
    L = _native.lib()
    buf = ctypes.create_string_buffer(1 << 22)
    nb = ctypes.c_size_t()
    P = low.prog_bytes()
    rc = L.sfg_jit_check(P, len(P), low.ins.ctypes.data, 10**6 * 8, buf, len(buf), ctypes.byref(nb))
    if dump:
        Path(dump).write_text(buf.value.decode())
    return rc, nb.value, buf.value.decode()


if __name__ == "__main__":
    names = sys.argv[1:] or ["dot"]
    assets = json.loads((REPO / "tests/golden/bench_assets.json").read_text())
    for n in names:
        if n in assets:
            m = harness_from_text(assets[n]["harness"], assets[n]["kernel"], f"{n}/harness.man")
        else:
            from paper_2603_05725_b200.workloads import load
            m = load(n)
        rc, nb, text = check(m, dump=f"/tmp/jit_{n}.cu")
        print(n, "rc", rc, "cubin", nb)
        if rc:
            print(text[:3000])
