"""Build libchunklab_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2604_10597_b200.build [--force] [--verbose]

The shared library is the product: the extern "C" ABI of include/chunklab_capi.h
over the CUDA kernels in csrc/.  cudart is linked statically so the .so only
needs the NVIDIA driver at run time.
"""
from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libchunklab_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def fingerprint() -> str:
    """sha256 of what determines the library's code: every source and header, the nvcc
    flags and the toolkit's version file.  nvcc's output bytes are not reproducible from
    build to build (embedded module ids), so measurements recorded against a build (the
    scan's ncu DRAM traffic, profiles/scan_traffic.json) are keyed to this instead."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join(ARCH + NVCC_FLAGS[:-2]).encode())  # flags without the absolute -I paths
    for f in sources() + headers():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    ver = os.path.join(os.path.dirname(os.path.dirname(nvcc())), "version.json")
    if os.path.exists(ver):
        with open(ver, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    hdrs = headers()
    objs = []
    nv = nvcc()
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            cmd = [nv, *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _newer(LIB, objs):
        cmd = [nv, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl",
               "-lrt"]  # NCCL is dlopen'ed by cl_collectives_nccl (no link dependency)
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print -Xptxas -v register/smem usage")
    args = ap.parse_args(argv)
    path = build(force=args.force, verbose=args.verbose, ptxas_verbose=args.ptxas)
    print(path)
    return 0


if __name__ == "__main__":
    sys.exit(main())
