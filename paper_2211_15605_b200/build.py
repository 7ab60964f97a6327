"""Build libmfx.so in-tree with nvcc for sm_100a (B200).

    python paper_2211_15605_b200/build.py [--force] [--verbose]

--fmad=false: no FMA contraction (DESIGN.md §3 arithmetic contract; fma() is
explicit).  -cudart static keeps the library independent of torch's cudart.
NCCL is dlopen'ed at run time (torch's libnccl.so.2), only its header is used.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libmfx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall",
    "-Xptxas", "-v" if os.environ.get("MFX_PTXAS_V") else "-O3",
    "-shared", "-cudart", "static",
    "-I" + os.path.join(ROOT, "include"),
    "-I/usr/include",
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "mfx.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO):
        so_t = os.path.getmtime(SO)
        if all(os.path.getmtime(p) <= so_t for p in deps()):
            return SO
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *sources(), "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(SO)
