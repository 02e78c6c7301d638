"""Build libcsplat variants with extra -D flags (tuning sweeps on the GPU box).

usage: python tools/variants.py name:-DFOO=1,-DBAR=2 [name2:...]
Writes variants/<name>.so; select one at run time with CSPLAT_LIB=variants/<name>.so.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200 import _build  # noqa: E402


def main():
    out = os.path.join(_build.ROOT, "variants")
    os.makedirs(out, exist_ok=True)
    procs = []
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition(":")
        flags = [d for d in defs.split(",") if d]
        srcs = [os.path.join(_build.CSRC, s) for s in _build.SOURCES]
        cmd = [_build.NVCC, *_build.nvcc_flags(flags), "-shared", "-o",
               os.path.join(out, name + ".so"), *srcs, "-lcudart"]
        procs.append((name, subprocess.Popen(cmd)))
    bad = [n for n, p in procs if p.wait() != 0]
    if bad:
        sys.exit("failed: " + " ".join(bad))


if __name__ == "__main__":
    main()
