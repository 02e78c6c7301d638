"""One C5 window iteration (64 keyframes x 500k, BatchedWindow, eager launches)
for an ncu launch list: `python tools/prof_c5.py [iters]`.  With
CSPLAT_SINGLE_STREAM unset the window still uses its two streams; ncu
serialises them, so compare per-kernel SUMS, not the wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11247_b200 import _build  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from paper_2403_11247_b200.window import gpu_window  # noqa: E402
from scenes import synth  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    _build.build()
    dev = torch.device("cuda:0")
    sc = synth.window_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    st.size_pairs(sc.views[0], views=sc.views)
    H, W = sc.cam["height"], sc.cam["width"]
    st.set_upstream(*(torch.tensor(a, device=dev)
                      for a in synth.upstream(np.random.default_rng(5), H, W)))
    win = gpu_window(st, sc.views, rank=0, world=1, reduce=False, batched=True)
    t0 = time.time()
    for _ in range(iters):
        win.run()
    torch.cuda.synchronize()
    win.check_capacity()
    pairs = win.vb["tile_range"][:, -1, 1].cpu().numpy().view("uint32")
    print("iters", iters, "s", round(time.time() - t0, 3), "max pairs per keyframe",
          int(pairs.max()), "n", st.n)


if __name__ == "__main__":
    main()
