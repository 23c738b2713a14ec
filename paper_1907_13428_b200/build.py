"""Build the in-tree sm_100a library paper_1907_13428_b200/lib/libfdg.so.

    python paper_1907_13428_b200/build.py [--force]

nvcc cross-compiles for sm_100a without a GPU; the built .so travels to GPU
boxes inside the repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libfdg.so")
SOURCES = ["fdg_kernels.cu", "fdg_api.cu", "fdg_pfa.cu"] + sorted(
    f for f in os.listdir(CSRC) if f.startswith("fdg_inst_") and f.endswith(".cu"))
HEADERS = [f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "--diag-suppress", "177"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "fdg.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every translation unit in parallel (nvcc -c), link libfdg.so."""
    from concurrent.futures import ThreadPoolExecutor
    lib = out or LIB
    if out is None and not defines and not force and not _stale():
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objdir = os.path.join(os.path.dirname(lib), "obj" + ("" if out is None else "_" + os.path.basename(lib)))
    os.makedirs(objdir, exist_ok=True)
    extra = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *extra, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    # python build.py [--force] [NAME -DDEF ...]: a variant library lib/libfdg_NAME.so
    if args:
        name, defs = args[0], [a[2:] for a in args[1:] if a.startswith("-D")]
        print(build(defines=defs, out=os.path.join(PKG, "lib", f"libfdg_{name}.so"), verbose=False))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
