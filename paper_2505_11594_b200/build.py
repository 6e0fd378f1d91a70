"""Build libsage3.so in-tree with nvcc for sm_100a (no torch extension machinery, no JIT cache).

    python -m paper_2505_11594_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsage3.so")
SOURCES = ["abi.cu", "quant.cu", "attn.cu", "attn_lazy.cu", "quant_i8.cu", "attn_i8.cu", "bwd_i8.cu"]
HEADERS = ["sm100.cuh", "attn_common.cuh", "internal.h", os.path.join("..", "..", "include", "sage3.h")]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-shared", "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libsage3.so (or `out`, with extra -D `defines`, for experiments)."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
    tmp = target + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
