"""Build libpobk.so in-tree (nvcc for sm_100a; host code with -ffp-contract=off).

    python paper_2401_00672_b200/build.py [--force]   (by path: importing the package loads the library)
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("POBK_BUILD_OUT", os.path.join(HERE, "libpobk.so"))  # development variants build elsewhere
BUILD = os.environ.get("POBK_BUILD_DIR", os.path.join(HERE, "_build"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [f"-DPOBK_K2_MAXJ={os.environ.get('POBK_K2_MAXJ', '24')}", "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
          "-I" + os.path.join(HERE, "..", "include")] + os.environ.get("POBK_EXTRA_FLAGS", "").split()

SOURCES = [
    "host/preprocess.cpp",
    "host/blocks.cpp",
    "capi.cpp",
    "cuda/vec_kernels.cu",
    "cuda/k1_launch.cu",
    "cuda/k1_multi.cu",
    "cuda/k3_smem.cu",
    "cuda/k2_wavefront.cu",
    "cuda/k4_cluster.cu",
    "cuda/k5_blocks.cu",
]
HEADERS = ["internal.h", "plan.h", "cuda/common.cuh", "../../include/pobk.h"]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_time = _newest([os.path.join(CSRC, h) for h in HEADERS])
    objs = []
    t0 = time.time()
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace("/", "_") + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_time):
            continue
        cmd = [NVCC] + COMMON + ARCH + ["-c", path, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if os.environ.get("POBK_PTXAS_V") else []
        if verbose:
            print("[build]", src, flush=True)
        subprocess.check_call(cmd)
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < _newest(objs):
        link = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", OUT + ".tmp"] + objs + ["-cudart", "static", "-lrt", "-lpthread", "-ldl"]
        subprocess.check_call(link)
        os.replace(OUT + ".tmp", OUT)
        if verbose:
            print(f"[build] linked {OUT} in {time.time() - t0:.1f}s", flush=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
