"""Build and bind the C-ABI library ``libsfg_b200.so`` (include/sfg.h).

The library is compiled in-tree for sm_100a with nvcc (no JIT cache, so the
built file travels to the GPU box with the repo snapshot).  Binding is plain
ctypes: raw device pointers, sizes and a cudaStream_t.  There is no fallback:
if the library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libsfg_b200.so"
HEADER = PKG.parent / "include" / "sfg.h"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static"]

EXPORTS = ("sfg_abi_version", "sfg_last_error", "sfg_program_create", "sfg_program_update",
           "sfg_program_destroy", "sfg_execute_smem_bytes", "sfg_plan", "sfg_mutate", "sfg_apply",
           "sfg_regen", "sfg_execute", "sfg_triage", "sfg_commit", "sfg_child_bytes", "sfg_compact",
           "sfg_scan_u32", "sfg_scan_u64", "sfg_layout_probe")


class NativeError(RuntimeError):
    pass


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [HEADER]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources())


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc, *NVCC_FLAGS, "-o", str(LIB), str(CSRC / "abi.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise NativeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    (PKG / "build_ptxas.log").write_text(res.stderr)
    if verbose:
        print(res.stderr)
    return LIB


_lib = None


def lib():
    """The loaded library (raises NativeError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        raise NativeError(f"{LIB} is not built; run __graft_entry__.build()")
    L = ctypes.CDLL(str(LIB))
    vp, sz, i32, i64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int64
    L.sfg_abi_version.restype = i32
    L.sfg_last_error.restype = ctypes.c_char_p
    L.sfg_program_create.argtypes = [vp, sz, vp, sz, vp, sz, vp, sz, vp, sz, vp, sz, vp, ctypes.POINTER(vp)]
    L.sfg_program_update.argtypes = [vp, vp, sz]
    L.sfg_program_destroy.argtypes = [vp]
    L.sfg_program_destroy.restype = None
    L.sfg_execute_smem_bytes.argtypes = [vp]
    L.sfg_execute_smem_bytes.restype = sz
    L.sfg_plan.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp]
    L.sfg_mutate.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp, vp]
    L.sfg_apply.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp]
    L.sfg_regen.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp, vp]
    L.sfg_execute.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.sfg_triage.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.sfg_commit.argtypes = [vp, vp, vp, vp]
    L.sfg_child_bytes.argtypes = [vp, vp, vp, i32, vp, vp]
    L.sfg_compact.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, ctypes.c_uint64, vp, vp, vp, vp, vp, vp]
    L.sfg_layout_probe.argtypes = [i32]
    L.sfg_layout_probe.restype = sz
    for f in ("sfg_scan_u32", "sfg_scan_u64"):
        getattr(L, f).argtypes = [vp, i64, i32, i32, vp, i32, i32, vp, vp, vp]
    for f in EXPORTS:
        if f not in ("sfg_abi_version", "sfg_last_error", "sfg_program_destroy", "sfg_execute_smem_bytes",
                     "sfg_layout_probe"):
            getattr(L, f).restype = i32
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().sfg_last_error().decode(errors="replace")
        raise NativeError(f"{what}: {msg}")


def loaded_path() -> str | None:
    return str(LIB) if _lib is not None else None


def env_summary() -> dict:
    return {"lib": str(LIB), "exists": LIB.exists(), "pid": os.getpid()}
