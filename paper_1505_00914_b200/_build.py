"""In-tree build of the native library (no JIT cache: the .so travels with
the repo snapshot to the GPU box).

    libchp_b200.so = the sm_100a kernels + C ABI (csrc/*.cu)
                   + the C++ drop-in of the reference entry points
                     (csrc/dropin/*.cpp over include/chp/*.hpp)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
# CHP_LIB_VARIANT (diagnostics): a separately built library, e.g. "bounds"
# (CHP_NVCC_EXTRA=-DCHP_BOUNDS=1: device-side index checks that trap) as
# lib/libchp_b200_bounds.so, loaded instead of the product library.
_VARIANT = os.environ.get("CHP_LIB_VARIANT", "")
LIB = os.path.join(LIBDIR, "libchp_b200%s.so" % (("_" + _VARIANT) if _VARIANT else ""))
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
                     "-I" + INCLUDE, "-I" + CSRC]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "dropin", "*.cpp")))


def headers() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
            + glob.glob(os.path.join(INCLUDE, "chp", "*.hpp")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(ROOT, "build", "obj" + (("_" + _VARIANT) if _VARIANT else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        # CHP_NVCC_EXTRA: instrumentation builds only (e.g. -DCHP_PHASE_TIMING=1, tools/phase_timing.py)
        cmd = [nvcc()] + NVCC_FLAGS + os.environ.get("CHP_NVCC_EXTRA", "").split() + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):  # host-only C++ over the C ABI
            cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++20", "-fPIC", "-Wall", "-I" + INCLUDE,
                   "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            print(out.decode())
        if p.returncode:
            failed.append(src)
    if failed:
        raise RuntimeError("nvcc failed: " + ", ".join(failed))
    tmp = LIB + ".tmp"
    subprocess.run([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-lpthread", "-ldl", "-lrt"],
                   check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
