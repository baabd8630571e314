"""Build the native code in-tree: libstablemerge.so for sm_100a (nvcc
cross-compiles without a GPU) and the oracle's liboracle.so (gcc).

    python build_native.py [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1202_6575_b200")
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libstablemerge.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(ROOT, "include", "stablemerge.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra_flags=None) -> str:
    """One object per translation unit (sm_common.cu + one abi_<key>.cu per key
    type), compiled in parallel, then linked into the shared library."""
    if out == LIB and extra_flags is None and not force and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objdir = os.path.join(ROOT, "build", "obj_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("SM_NVCC_EXTRA", "").split() if extra_flags is None else list(extra_flags)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *COMPILE_FLAGS, *extra, *inc, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs])
    return out


DEBUG_LIB = os.path.join(LIBDIR, "libstablemerge_debug.so")


def build_debug(force: bool = False) -> str:
    """The SM_DEBUG build (device-side store-range checks and K2's output
    coverage counters, include/stablemerge.h sm_debug_cover): a separate
    library beside the product one, loaded only when asked for
    (SM_LIB_PATH)."""
    if not force and os.path.exists(DEBUG_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(DEBUG_LIB)
                                                       for d in deps()):
        return DEBUG_LIB
    return build(out=DEBUG_LIB, extra_flags=["-DSM_DEBUG"])


def build_oracle() -> str:
    """The CPU oracle (test infrastructure) -- building the checker is not using it."""
    sys.path.insert(0, ROOT)
    import oracle
    return oracle.build()


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
    if "--debug" in sys.argv:
        print(build_debug(force=True))
    print(build_oracle())
