"""Build libfmmlu.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Usage: python -m paper_2201_07325_b200.build   (or build() from __graft_entry__)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.environ.get("FMMLU_LIBDIR") or os.path.join(HERE, "lib")  # override: experiment builds
LIB = os.path.join(LIBDIR, "libfmmlu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I", os.path.join(HERE, "..", "include")] + os.environ.get("FMMLU_NVCC_EXTRA", "").split()
CU = ["fmmlu.cu", "kernels.cu", "gemm.cu", "rootlu.cu", "devtree.cu"]
CPP = ["tree.cpp"]
CXX = os.environ.get("CXX", "g++")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def sources():
    return [os.path.join(CSRC, f) for f in CU + CPP] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))
    ] + [os.path.join(HERE, "..", "include", "fmmlu.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def cu(f):
        o = os.path.join(objdir, f + ".o")
        out = _run([NVCC, *ARCH, *COMMON, "-Xptxas", "-v" if verbose else "-O3", "-c",
                    os.path.join(CSRC, f), "-o", o])
        if verbose:
            sys.stderr.write(out)
        return o

    def cpp(f):
        o = os.path.join(objdir, f + ".o")
        _run([CXX, "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-c", os.path.join(CSRC, f), "-o", o])
        return o

    with ThreadPoolExecutor(max_workers=len(CU) + len(CPP)) as ex:  # one compiler process per source
        futs = [ex.submit(cu, f) for f in CU] + [ex.submit(cpp, f) for f in CPP]
        objs = [f.result() for f in futs]
    _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-Xcompiler", "-pthread"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
