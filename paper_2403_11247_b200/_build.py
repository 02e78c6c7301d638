"""Build libcsplat.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcsplat.so")
SOURCES = ["api.cu", "project.cu", "bin.cu", "render_fwd.cu", "render_bwd.cu", "chain.cu", "rvq.cu",
           "prune.cu", "loss.cu", "rvq_update.cu", "ba.cu", "record_tmap.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nvcc_flags(extra=()):
    return ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
            "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "--expt-relaxed-constexpr",
            "-I" + os.path.join(ROOT, "include"), *extra]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("common.cuh", "bin_dev.cuh", "quad.cuh", "composite.cuh")] + \
        [os.path.join(ROOT, "include", "csplat.h")]
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB
    cmd = [NVCC, *nvcc_flags(["-Xptxas", "-v"] if verbose else []), "-shared", "-o", LIB, *srcs,
           "-lcudart"]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
