"""Compile liblofp.so (and the bench's FP64 peak probe) in-tree for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("lofp_kernels.cu", "lofp_contract.cu", "lofp_host.cpp")]
HEADERS = [os.path.join(CSRC, "lofp_internal.h"), os.path.join(ROOT, "include", "lofp.h")]
LIB = os.path.join(HERE, "liblofp.so")
PEAK_SRC = os.path.join(CSRC, "fp64_peak.cu")
PEAK_LIB = os.path.join(HERE, "libfp64peak.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-ldl"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _compile(out, sources, deps, force, verbose):
    newest = max(os.path.getmtime(p) for p in sources + deps)
    if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
        tmp = out + f".tmp{os.getpid()}"
        cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-o", tmp] + sources
        subprocess.check_call(cmd)
        os.replace(tmp, out)
    return out


DEBUG_LIB = os.path.join(HERE, "liblofp_debug.so")


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """liblofp.so (and the FP64 peak probe); debug=True also builds liblofp_debug.so, the
    same sources with device-side bounds checks (-DLOFP_DEBUG), loaded when LOFP_LIB
    points at it."""
    _compile(PEAK_LIB, [PEAK_SRC], [], force, False)
    if debug:
        global NVCC_FLAGS
        saved = NVCC_FLAGS
        NVCC_FLAGS = saved + ["-DLOFP_DEBUG"]
        try:
            _compile(DEBUG_LIB, SOURCES, HEADERS, force, verbose)
        finally:
            NVCC_FLAGS = saved
    return _compile(LIB, SOURCES, HEADERS, force, verbose)
