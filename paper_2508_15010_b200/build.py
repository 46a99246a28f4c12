"""Build libtoast.so in-tree (paper_2508_15010_b200/lib/) for sm_100a.

    python -m paper_2508_15010_b200.build [--force]

Kernels: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false.
Host code: g++ -O2 -ffp-contract=off (the search's UCT arithmetic and the
baseline score are plain IEEE double, evaluated in a fixed order).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "lib", "libtoast.so")
INC = os.path.join(os.path.dirname(HERE), "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = GENCODE + ["-O3", "-lineinfo", "-std=c++20", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
                      f"-I{INC}", f"-I{SRC}"]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", f"-I{CUDA}/include", f"-I{INC}", f"-I{SRC}"]

SOURCES = ["ir.cpp", "analysis.cpp", "lower.cpp", "search.cpp", "abi.cpp", "kernels.cu"]
HEADERS = ["toast_internal.h"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, obj: str = OBJ, extra=()) -> str:
    """extra: additional nvcc flags for the kernels (used by scripts/kernel_sweep.py)."""
    global LIB, OBJ
    saved = (LIB, OBJ)
    LIB, OBJ = lib, obj
    try:
        return _build(force, verbose, list(extra))
    finally:
        LIB, OBJ = saved


def _build(force: bool, verbose: bool, extra) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = [os.path.join(SRC, h) for h in HEADERS] + [os.path.join(INC, "toast.h")]
    objs = []
    for s in SOURCES:
        src = os.path.join(SRC, s)
        obj = os.path.join(OBJ, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            if s.endswith(".cu"):
                cmd = [NVCC] + CU_FLAGS + extra + ["-c", src, "-o", obj]
            else:
                cmd = ["g++"] + CXX_FLAGS + ["-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
    if force or _newer(LIB, objs):
        cmd = [NVCC] + GENCODE + ["-shared", "-o", LIB] + objs + ["-Xcompiler", "-fPIC", "-lpthread"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return LIB


LIB_CHECKED = os.path.join(HERE, "lib", "libtoast_checked.so")


def build_checked(force: bool = False, verbose: bool = False) -> str:
    """The checked library (kernels.cu TOAST_CHECKED: shared-memory bounds and
    table-index checks, dead-region poisoning, randomised barrier timing) —
    test infrastructure for the race / bounds evidence; the
    product path never loads it."""
    return build(force=force, verbose=verbose, lib=LIB_CHECKED, obj=os.path.join(HERE, "build", "checked"),
                 extra=["-DTOAST_CHECKED=1"])


LIB_MUTANT = os.path.join(HERE, "lib", "libtoast_checked_mutant.so")


def build_checked_mutant(force: bool = False, verbose: bool = False) -> str:
    """The checked library with one barrier removed (TOAST_CHK_MUTANT: warps
    read the decode results without waiting for them) — the planted race the
    checker must catch (tests/test_gpu_parity.py)."""
    return build(force=force, verbose=verbose, lib=LIB_MUTANT, obj=os.path.join(HERE, "build", "mutant"),
                 extra=["-DTOAST_CHECKED=1", "-DTOAST_CHK_MUTANT=1"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv, verbose=True))
