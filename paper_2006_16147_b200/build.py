"""Build the product library libamg_b200.so in-tree for sm_100a.

g++ compiles the host setup with -ffp-contract=off (canonical arithmetic
contract C1); nvcc compiles the device code and the ABI for
`-gencode arch=compute_100a,code=sm_100a` only.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# AMG_BUILD_VARIANT=<name> (experiments only): extra -D flags from AMG_BUILD_DEFS, a separate build
# directory and libamg_b200_<name>.so, loaded when AMG_LIB_PATH points at it (_abi.py)
VARIANT = os.environ.get("AMG_BUILD_VARIANT", "")
DEFS = os.environ.get("AMG_BUILD_DEFS", "").split() if VARIANT else []
BUILD = os.path.join(PKG, "_build" + ("_" + VARIANT if VARIANT else ""))
LIB = os.path.join(PKG, "libamg_b200" + ("_" + VARIANT if VARIANT else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]

SOURCES_CXX = [os.path.join(CSRC, "setup", "setup.cpp"), os.path.join(CSRC, "setup", "partition.cpp"),
               os.path.join(CSRC, "setup", "dist_setup.cpp")]
SOURCES_CU = [os.path.join(CSRC, "amg_api.cu")]
# the GPU setup must follow the canonical arithmetic contract C1 (no FMA contraction)
SOURCES_CU_NOFMA = [os.path.join(CSRC, "setup", "setup_gpu.cu")]
HEADERS = [os.path.join(CSRC, "kernels.cuh"), os.path.join(CSRC, "setup", "setup.hpp"),
           os.path.join(CSRC, "setup", "partition.hpp"), os.path.join(CSRC, "setup", "dist_setup.hpp"),
           os.path.join(ROOT, "include", "amg_b200.h")]


def _run(cmd):
    print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in SOURCES_CXX:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + HEADERS):
            _run(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off",
                  "-Wall", "-c", src, "-o", obj])
        objs.append(obj)
    for src in SOURCES_CU + SOURCES_CU_NOFMA:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + HEADERS):
            cmd = [NVCC] + ARCH + DEFS + ["-O3", "-lineinfo", "-std=c++17", "-I", os.path.join(_nccl_dir(), "include"),
                                   "-Xcompiler",
                                   "-fPIC,-fopenmp,-ffp-contract=off", "-c", src, "-o", obj]
            if src in SOURCES_CU_NOFMA:
                cmd[1:1] = ["--fmad=false", "-prec-div=true", "-prec-sqrt=true"]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(obj)
    if force or _stale(LIB, objs):
        nlib = os.path.join(_nccl_dir(), "lib")
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-lgomp", "-L", nlib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nlib}", "-Xlinker", "-z,defs"])
    return LIB


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
