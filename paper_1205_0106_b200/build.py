"""Builds libqmcg.so (CUDA kernels + C ABI + C++ drop-in) in-tree for sm_100a.

The library is compiled straight with nvcc / g++ (no JIT cache), so the built
file travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libqmcg.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["kernels.cu"]
CXX_SOURCES = ["api.cpp", "dropin.cpp"]
HEADERS = ["qmcg_internal.h"]


def _run(cmd: list[str]) -> None:
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out.stdout + out.stderr)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), lib: str = LIB,
          build_dir: str = BUILD) -> str:
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(INCLUDE, "qmcg.h"), os.path.join(INCLUDE, "qmc_b200", "qmc.hpp")]
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
                   "-I", INCLUDE, "-I", CSRC, "-I", "/usr/local/cuda/include", *[f"-D{d}" for d in defines],
                   "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd))
        _run(cmd)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
