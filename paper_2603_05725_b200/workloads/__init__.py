"""Synthetic fuzz targets for the BASELINE.json configs (SIR + harness text in
the reference's own formats, so the reference and the oracle can run them)."""

from pathlib import Path

HERE = Path(__file__).resolve().parent


def manifest_path(name: str) -> Path:
    return HERE / f"{name}.man"


def load(name: str):
    from ..manifest import load_harness
    return load_harness(manifest_path(name))
