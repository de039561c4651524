"""Builds the in-tree shared library libibm_b200.so for sm_100a with nvcc.

Flags: --fmad=false and host -ffp-contract=off implement the arithmetic
contract of DESIGN.md §3 (R13, no FMA contraction); -lineinfo for ncu source
views; linked against NCCL for the slab-decomposed multi-GPU path.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libibm_b200.so")
SOURCES = ["kernels.cu", "sor.cu", "sor_wf.cu", "sor_tb.cu", "api.cu"]
HEADERS = ["ibm_internal.h", "sor_common.cuh", os.path.join("..", "..", "include", "ibm.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2,-fvisibility=hidden",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("IBM_NVCC_DEFS", "").split()  # tuning experiments only (-DNAME=value)
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            sys.stderr.write(out.stdout + out.stderr)
            raise RuntimeError("nvcc failed for %s" % src)
        if verbose:
            sys.stderr.write(out.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lnccl", "-cudart", "static"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
