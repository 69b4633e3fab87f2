"""Build the sm_100a shared library in-tree (no JIT cache: the .so travels to
the GPU box with the repo snapshot)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libdcopf_dual.so")
SOURCES = [os.path.join(CSRC, "dcopf_dual.cu"), os.path.join(CSRC, "schedule.cpp"),
           os.path.join(CSRC, "split_schedule.cpp"), os.path.join(CSRC, "cluster.cpp"), os.path.join(CSRC, "ptdf.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("dual_kernels.cuh", "fp64_fast.cuh", "sweep_kernel.cuh", "schedule.h", "schedule_detail.h", "cluster.h",
                                              "cluster_kernel.cuh", "ptdf.h")] + [
    os.path.join(ROOT, "include", "dcopf_dual.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",             # no FMA contraction: same rounding as the oracle (reading A-19)
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(p) <= t for p in DEPS):
            return LIB
    # one object per source, compiled in parallel, then one shared-library link
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc()] + flags + ["-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs, log = [], ""
    for obj, pr in procs:
        out, errs = pr.communicate()
        log += errs
        if pr.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + out + errs)
        objs.append(obj)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp"] + objs
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(log)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
