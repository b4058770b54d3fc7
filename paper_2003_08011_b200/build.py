"""Builds the in-tree extension ``libcstress_b200.so`` for sm_100a.

nvcc cross-compiles without a GPU, so this runs anywhere the CUDA 12.9
toolchain is installed.  The shared library is the product: the C-ABI declared
in ``include/cstress_b200.h`` plus the C++ host layer.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcstress_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["cstress_b200.cu", "synth.cpp", "model_io.cpp"]


def _sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def _deps():
    out = []
    for d, _, files in os.walk(CSRC):
        out += [os.path.join(d, f) for f in files]
    out.append(os.path.join(ROOT, "include", "cstress_b200.h"))
    out.append(os.path.abspath(__file__))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *_sources(), "-o", LIB + ".tmp",
           "-lpthread", "-ldl"]
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(LIB + ".tmp", LIB)
    return LIB


CPP_TEST = os.path.join(ROOT, "tests", "cpp", "test_b200_api.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_b200_api")


def build_cpp_test() -> str:
    """The C++ host-layer test program (include/cstress_b200.hpp)."""
    build()
    if (os.path.exists(CPP_TEST_BIN) and os.path.getmtime(CPP_TEST_BIN) >= max(
            os.path.getmtime(p) for p in [CPP_TEST, LIB, os.path.join(ROOT, "include", "cstress_b200.hpp")])):
        return CPP_TEST_BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), CPP_TEST,
                    "-o", CPP_TEST_BIN, "-L", HERE, "-lcstress_b200", f"-Wl,-rpath,{HERE}"], check=True)
    return CPP_TEST_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
