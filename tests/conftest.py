import json
import os
import sys
from functools import lru_cache
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: longer CPU parity runs")


@lru_cache(maxsize=None)
def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


def bench_names():
    return sorted(golden("bench_assets.json"))


@lru_cache(maxsize=None)
def bench_manifest(name: str, variant: str | None = None):
    from paper_2603_05725_b200.manifest import harness_from_text
    a = golden("bench_assets.json")[name]
    if variant is not None and "harness" in a["variants"][variant]:
        v = a["variants"][variant]
        return harness_from_text(v["harness"], v["kernel"], f"{name}/{variant}/harness.man")
    return harness_from_text(a["harness"], a["kernel"], f"{name}/harness.man")


def trigger_ops(name: str, variant: str):
    from paper_2603_05725_b200.testcase import MutationOp
    text = golden("bench_assets.json")[name]["variants"][variant]["trigger"]
    lines = [l.strip() for l in text.splitlines() if l.strip() and not l.startswith("#")]
    expected = next(l[6:] for l in lines if l.startswith("class="))
    return expected, tuple(MutationOp.decode(l) for l in lines if l.startswith("mut "))


def workload_manifest(stem: str):
    from paper_2603_05725_b200.manifest import load_harness
    return load_harness(REPO / "paper_2603_05725_b200" / "workloads" / f"{stem}.man")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


WORKLOADS = ("matmul", "vadd", "ctxchain", "structcfg")


def workload_case(stem: str):
    """(manifest, campaign kwargs, round size, iterations) of a golden workload
    campaign (tests/golden/make_golden.py workloads)."""
    from paper_2603_05725_b200.testcase import parse_testcase
    m = workload_manifest(stem)
    if stem == "structcfg":
        seeds = tuple(parse_testcase(t)[0] for t in golden("ref_workloads.json")[stem]["seeds"])
        return m, {"extra_seeds": seeds, "fanout": 8}, 1600, 3200
    return m, {}, 100, 300
