"""Build the in-tree shared library libtn_b200.so (C ABI in include/tn.h).

Host C++ (network builder, order finder) is compiled with -ffp-contract=off so that
every floating-point decision of the order search is a plain IEEE-754 operation;
device code is compiled for sm_100a only.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libtn_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SRCS = ["host/network.cpp", "host/order.cpp"]
CUDA_SRCS = ["runtime.cu"]
DEPS = ["host/tn_host.hpp", "device/common.cuh", "device/small.cu", "device/gemm_tc.cu", "device/zgemm.cu", "device/skinny.cu",
        os.path.join("..", "..", "include", "tn.h")]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(s) and os.path.getmtime(s) > t for s in src_list)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} exit {r.returncode}")
    return r.stdout + r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    deps = [os.path.join(CSRC, d) for d in DEPS]
    objs = []
    for s in HOST_SRCS:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, os.path.basename(s) + ".o")
        if force or _newer([src] + deps, obj):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-pthread", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                  *inc, "-c", src, "-o", obj])
        objs.append(obj)
    for s in CUDA_SRCS:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, os.path.basename(s) + ".o")
        if force or _newer([src] + deps, obj):
            out = _run([NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v",
                        *os.environ.get("TN_NVCC_EXTRA", "").split(),
                        "-Xcompiler", "-fPIC,-ffp-contract=off", *inc, "-c", src, "-o", obj])
            if verbose:
                sys.stdout.write(out)
            with open(os.path.join(BUILD, os.path.basename(s) + ".ptxas.txt"), "w") as f:
                f.write(out)
        objs.append(obj)
    if force or _newer(objs, LIB):
        _run([NVCC, "-shared", *ARCH, "-o", LIB, *objs, "-lcudart", "-Xcompiler", "-pthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
