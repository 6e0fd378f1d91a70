"""Build libsage3.so in-tree with nvcc for sm_100a (no torch extension machinery, no JIT cache).

    python -m paper_2505_11594_b200.build [--force] [--verbose]

Each source is compiled to a relocatable object in parallel (one nvcc per file), then linked into one
shared library.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsage3.so")
OBJ_CACHE = os.path.join(os.environ.get("TMPDIR", "/tmp"), "sage3_obj_cache")  # outside the repo snapshot
SOURCES = ["abi.cu", "quant.cu", "attn.cu", "attn3.cu", "attn_lazy.cu", "quant_i8.cu", "attn_i8.cu", "bwd_i8.cu"]
HEADERS = ["sm100.cuh", "attn_common.cuh", "internal.h", os.path.join("..", "..", "include", "sage3.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC"]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=(), only=None) -> str:
    """Compile libsage3.so (or `out`, with extra -D `defines`, for experiments; `only`: the sources the defines
    apply to, the others built with the default flags)."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
    tmpdir = tempfile.mkdtemp(prefix="sage3build")
    try:
        base = [*NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-I", os.path.join(ROOT, "include"), "-I", CSRC]
        flags = lambda src: base + ([f"-D{d}" for d in defines] if only is None or src in only else [])

        hdr = b"".join(open(os.path.join(CSRC, h), "rb").read() for h in HEADERS)

        def obj(src):
            # objects are cached by content (source, headers, flags) under build/obj: variant builds for A/B runs
            # only recompile the files their -D flags can change
            common = flags(src)
            key = hashlib.sha1(open(os.path.join(CSRC, src), "rb").read() + hdr + " ".join(common).encode()).hexdigest()
            cached = os.path.join(OBJ_CACHE, f"{src[:-3]}-{key[:16]}.o")
            if not os.path.exists(cached):
                o = os.path.join(tmpdir, src.replace(".cu", ".o"))
                subprocess.run([_nvcc(), *common, "-c", os.path.join(CSRC, src), "-o", o], check=True)
                os.makedirs(OBJ_CACHE, exist_ok=True)
                shutil.copyfile(o, cached + ".tmp")
                os.replace(cached + ".tmp", cached)
            return cached

        with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            objs = list(ex.map(obj, SOURCES))
        tmp = target + f".tmp{os.getpid()}"
        subprocess.run([_nvcc(), *ARCH, "-shared", "-o", tmp, *objs], check=True)
        os.replace(tmp, target)
    finally:
        shutil.rmtree(tmpdir, ignore_errors=True)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
