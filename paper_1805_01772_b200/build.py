"""Build libcf.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcf.so")
# profiling build (driver region profiler + per-instance timing compiled in): tools/ only
LIB_PROF = os.path.join(HERE, "libcf_prof.so")
SOURCES = ["ir.cpp", "autodiff.cpp", "capi.cpp", "compiler.cpp", "runtime.cu", "debug.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-diag-suppress", "177,550"]


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp", ".h", ".cuh"))] + \
        [os.path.join(HERE, "..", "include", f) for f in ("cf.h", "cf_debug.h")] + [__file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    lib = LIB_PROF if profile else LIB
    if not force and not _stale(lib):
        return lib
    # one builder at a time (e.g. every rank of a torchrun job): the others wait, then find
    # the library fresh
    import fcntl
    os.makedirs(os.path.join(CSRC, "build"), exist_ok=True)
    with open(os.path.join(CSRC, "build", ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not _stale(lib):
            return lib
        return _build_locked(lib, force, verbose, profile)


def _build_locked(lib: str, force: bool, verbose: bool, profile: bool) -> str:
    tag = "_prof" if profile else ""
    objs = []
    # headers (and this script) invalidate every object; a source only its own
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + \
        [os.path.join(HERE, "..", "include", f) for f in ("cf.h", "cf_debug.h")] + [__file__]
    t_hdr = max(os.path.getmtime(p) for p in hdrs if os.path.exists(p))
    for src in SOURCES:
        obj = os.path.join(CSRC, "build" + tag, src + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        objs.append(obj)
        if not force and os.path.exists(obj) and \
                os.path.getmtime(obj) > max(t_hdr, os.path.getmtime(os.path.join(CSRC, src))):
            continue
        cmd = [NVCC, *FLAGS, *(["-DCF_PROFILE"] if profile else []), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    tmp = lib + ".tmp"
    subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", tmp, "-lcudart"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
