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
SOURCES = ["cstress_b200.cu", "train_f64.cu", "synth.cpp", "model_io.cpp"]


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


OBJ_DIR = os.path.join(HERE, "build")


def _obj(src):
    return os.path.join(OBJ_DIR, os.path.basename(src) + ".o")


def _obj_stale(src) -> bool:
    """An object is stale when its source or any header it included (the
    nvcc -MD dependency file) is newer, or this build script changed."""
    o, d = _obj(src), _obj(src) + ".d"
    if not (os.path.exists(o) and os.path.exists(d)):
        return True
    t = os.path.getmtime(o)
    deps = [src, os.path.abspath(__file__)]
    text = open(d).read().replace("\\\n", " ")
    for tok in text.split(":", 1)[-1].split():
        deps.append(tok)
    return any((not os.path.exists(p)) or os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each source to an object (in parallel, incrementally via the
    -MD dependency files) and link libcstress_b200.so."""
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if verbose else "-O3",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    todo = [s for s in _sources() if force or _obj_stale(s)]

    def compile_one(src):
        subprocess.run([*common, "-MD", "-MF", _obj(src) + ".d", "-c", src, "-o", _obj(src)], check=True, cwd=CSRC)

    with ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    subprocess.run([NVCC, *ARCH, "--shared", "-Xcompiler", "-fPIC", *[_obj(s) for s in _sources()],
                    "-o", LIB + ".tmp", "-lpthread", "-ldl"], check=True, cwd=CSRC)
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
