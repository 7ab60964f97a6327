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
] + os.environ.get("MFX_EXTRA_NVCC_FLAGS", "").split()


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "mfx.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO):
        so_t = os.path.getmtime(SO)
        if all(os.path.getmtime(p) <= so_t for p in deps()):
            return SO
    # one object per translation unit, compiled in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor
    odir = os.path.join(HERE, "build")
    os.makedirs(odir, exist_ok=True)
    compile_flags = [f for f in FLAGS if f not in ("-shared",)]

    def compile_one(src):
        obj = os.path.join(odir, os.path.basename(src) + f".{os.getpid()}.o")
        cmd = [NVCC, *compile_flags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
           "-o", tmp, *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(SO)
