"""Build libperm.so in-tree: host C++ (planner, codegen, NVRTC runtime) and the
fixed sm_100a reduction kernels, compiled with nvcc for sm_100a only.

    python -m paper_2501_15126_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libperm.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SOURCES = ["matrix.cpp", "codegen.cpp", "planner.cpp", "runtime.cpp", "plan_io.cpp", "collective.cpp", "reduce.cu", "probe.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [
        os.path.join(CSRC, "perm_internal.h"), os.path.join(CSRC, "plan_state.h"), os.path.join(CSRC, "rt_internal.h"), os.path.join(ROOT, "include", "perm.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    nvcc = os.path.join(CUDA, "bin", "nvcc")
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-O3", "-std=c++17", "-lineinfo", *ARCH, "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-o", tmp, "-cudart", "static", "-L" + os.path.join(CUDA, "lib64"), "-lnvrtc", "-ldl",
           "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
