"""CPU calibration (build container): the oracle port (oracle/loop.batched_loop)
against the REAL reference's own functions driven under the same batched-round
contract (tests/golden/make_golden.batched), on the same inputs -- the first N
inputs of the bench workload's round 1 (C2 matmul, master_seed 11, R = 262,144;
records are prefix-consistent).  One process each, same host.
Usage: python tools/cpu_calibration.py [N]"""
import platform
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests" / "golden"))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return platform.processor()


import make_golden as mg  # noqa: E402  (imports the reference from /root/reference)
from oracle.loop import batched_loop  # noqa: E402
from paper_2603_05725_b200.workloads import load  # noqa: E402

m_ref = mg.rc.load_harness(REPO / "paper_2603_05725_b200" / "workloads" / "matmul.man")
t0 = time.perf_counter()
ref = mg.batched(m_ref, master_seed=11, iterations=N, round_size=262144)
t_ref = time.perf_counter() - t0
t0 = time.perf_counter()
port = batched_loop(load("matmul"), master_seed=11, iterations=N, round_size=262144)
t_port = time.perf_counter() - t0
import hashlib  # noqa: E402
from paper_2603_05725_b200.testcase import serialize_testcase  # noqa: E402
same = [r["child"] for r in ref["records"]] == [
    hashlib.sha256(serialize_testcase(r["child"], with_id=False).encode()).hexdigest()[:32] for r in port.records]
print(f"host: {cpu_model()}, {platform.python_implementation()} {platform.python_version()}, 1 process each")
print(f"inputs: the first {N} of C2 round 1 (matmul, master_seed 11, R=262144); identical children: {same}")
print(f"reference functions (batched contract): {t_ref:.1f} s -> {N / t_ref:.0f} execs/s")
print(f"oracle port (batched contract):         {t_port:.1f} s -> {N / t_port:.0f} execs/s")
print(f"port / reference speed ratio: {t_ref / t_port:.2f}")
