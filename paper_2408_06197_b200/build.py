"""Build the sm_100a CUDA library in-tree: paper_2408_06197_b200/_lib/liblancelot_b200.so.

nvcc cross-compiles without a GPU; the .so travels to the B200 box with the
repository snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "liblancelot_b200.so")
SOURCES = ["engine.cu"]
# every header engine.cu includes (globbed, so a new .cuh cannot be missed)
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "lancelot_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


CPP_DRIVER = os.path.join(OUT_DIR, "server_round")
CPP_SRC = os.path.join(os.path.dirname(HERE), "tests", "cpp", "server_round.cpp")


def build_cpp_driver(verbose: bool = False) -> str:
    """The C++ mirror (include/lancelot_b200.hpp) exercised as a reference
    caller would link it; used by tests/test_cpp_mirror.py."""
    hdrs = [os.path.join(os.path.dirname(HERE), "include", h)
            for h in ("lancelot_b200.h", "lancelot_b200.hpp")]
    if os.path.exists(CPP_DRIVER) and all(
            os.path.getmtime(CPP_DRIVER) > os.path.getmtime(x) for x in hdrs + [CPP_SRC, LIB]):
        return CPP_DRIVER
    cmd = ["g++", "-std=c++17", "-O2", "-pthread", "-I", os.path.join(os.path.dirname(HERE), "include"),
           CPP_SRC, "-o", CPP_DRIVER, "-L", OUT_DIR, "-llancelot_b200", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return CPP_DRIVER


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        build_cpp_driver(verbose)
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists("/usr/local/cuda/bin/nvcc") and nvcc == "nvcc":
        pass
    elif nvcc == "nvcc":
        nvcc = "/usr/local/cuda/bin/nvcc"
    tmp = LIB + ".tmp"
    cmd = [nvcc] + NVCC_FLAGS + ["-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    build_cpp_driver(verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
