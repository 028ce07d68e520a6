"""Builds libeeb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "eeb200.cu"), os.path.join(HERE, "csrc", "gemm.cu"),
           os.path.join(HERE, "csrc", "synth.cpp")]
HEADERS = [os.path.join(ROOT, "include", "eeb200.h")] + sorted(
    glob.glob(os.path.join(HERE, "csrc", "*.cuh")))
LIB = os.path.join(HERE, "libeeb200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    return shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit in parallel, then link the shared library."""
    if not force and not needs_build():
        return LIB
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off"]
    if verbose:
        flags.append("-Xptxas=-v")
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(HERE, "csrc", os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([nvcc(), *flags, "-c", "-o", obj, src]))
    if any(p.wait() != 0 for p in procs):
        raise subprocess.CalledProcessError(1, "nvcc")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs], check=True)
    os.replace(LIB + ".tmp", LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
