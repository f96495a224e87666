"""Builds librnnwave_sm100.so in-tree (paper_1604_01946_b200/lib/) with nvcc for sm_100a.

The .so is git-ignored but travels to the GPU box with the gpurun snapshot, so the box
never compiles anything. Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "librnnwave_sm100.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-shared", "-cudart", "static"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "rnnwave_sm100.h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    """Each kernel family is its own translation unit (csrc/kernels_*.cu + runtime.cu), compiled
    to objects in parallel and linked into one shared library."""
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    cu = [s for s in sources() if s.endswith(".cu")]
    compile_flags = [f for f in FLAGS if f not in ("-shared",)]
    procs, objs = [], []
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *compile_flags, "-c", "-I", os.path.join(ROOT, "include"), "-o", obj, src]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log_txt, failed = "", False
    for cmd, pr in procs:
        out, err = pr.communicate()
        log_txt += " ".join(cmd) + "\n" + out + err
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(err[-8000:])
    tmp = LIB + ".tmp"
    if not failed:
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", "-o", tmp, *objs]
        out = subprocess.run(cmd, capture_output=True, text=True)
        log_txt += " ".join(cmd) + "\n" + out.stdout + out.stderr
        if out.returncode != 0:
            failed = True
            sys.stderr.write(out.stderr[-8000:])
    log = os.path.join(LIBDIR, "build.log")
    with open(log, "w") as f:
        f.write(log_txt)
    if failed:
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, LIB)
    if verbose:
        print(log_txt[-4000:])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
