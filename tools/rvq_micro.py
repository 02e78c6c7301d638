"""Time csplat_rvq_assign alone on the C2 (200k, 75% kept) and C4 (1M) shapes:
python tools/rvq_micro.py [lib.so ...] (CUDA events, 20 reps, L2 not flushed).
Tuning builds with -DCSPLAT_RVQF_STATS also report the filter's fallback rate."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from scenes import synth  # noqa: E402


def run(libpath):
    os.environ["CSPLAT_LIB"] = libpath
    import importlib
    from paper_2403_11247_b200 import csplat as cs
    importlib.reload(cs)
    dev = torch.device("cuda:0")
    out = {}
    only = os.environ.get("RVQ_ONLY")  # e.g. "c4_log_scale" (ncu captures)
    for name, sc in [("c2", synth.replica_scene(0)), ("c4", synth.scannet_scene(0))]:
        if only and not only.startswith(name):
            continue
        keep = sc.mask > -4.59511995
        for attr, key in [("log_scale", "scale_codes"), ("quat", "rot_codes")]:
            if only and only != f"{name}_{attr}":
                continue
            x = torch.tensor(np.ascontiguousarray(getattr(sc, attr)[:, keep] if name == "c2"
                                                  else getattr(sc, attr)), device=dev)
            codes = torch.tensor(sc.codebook[key], device=dev)
            for _ in range(3):
                cs.rvq_assign(x, codes)
            st = ctypes.c_ulonglong * 2
            buf = st()
            f = getattr(cs.lib(), "csplat_debug_rvqf_stats", None)
            if f:
                f(buf)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                cs.rvq_assign(x, codes)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            rate = None
            if f:
                f(buf)
                rate = buf[1] / max(1, buf[0] + buf[1])
            out[f"{name}_{attr}"] = (round(us, 1), rate)
    print(os.path.basename(libpath), out, flush=True)


if __name__ == "__main__":
    for p in sys.argv[1:] or [os.path.join(os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))), "paper_2403_11247_b200", "libcsplat.so")]:
        run(p)
