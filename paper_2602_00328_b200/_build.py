"""Build libharvest_b200.so in-tree with nvcc for sm_100a.

The library is a plain C ABI (include/harvest_b200.h) with the CUDA runtime
linked statically, so it loads on a CPU-only machine (driver entry points are
resolved lazily) and travels to the GPU box inside the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "libharvest_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
SOURCES = ["hv_kernels.cu", "hv_ffn.cu", "hv_attn.cu", "hv_moe.cu", "hv_pool.cpp", "hv_segalloc.cpp", "hv_place.cpp"]
GENCODE = "arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the Harvest data plane has no CPU fallback")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, s) for s in SOURCES]
    deps += [os.path.join(CSRC, "hv_common.h"), os.path.join(REPO_DIR, "include", "harvest_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    cmd = [
        nvcc(), "-O3", "-std=c++17", "-gencode", GENCODE, "-lineinfo",
        "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-cudart", "static",
        "-I", os.path.join(REPO_DIR, "include"),
        "-o", tmp,
    ] + [os.path.join(CSRC, s) for s in SOURCES] + ["-ldl", "-lrt", "-lpthread"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
