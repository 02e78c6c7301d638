"""One batched C5 window iteration (for ncu launch lists): python tools/c5_batched_once.py [K]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from paper_2403_11247_b200.window import gpu_window  # noqa: E402
from scenes import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda:0")
sc = synth.window_scene(0)
views = sc.views[:K]
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
st.size_pairs(views[0], views=views[1:])
H, W = sc.cam["height"], sc.cam["width"]
st.set_upstream(*(torch.tensor(a, device=dev) for a in synth.upstream(np.random.default_rng(5), H, W)))
win = gpu_window(st, views, rank=0, world=1, batched=True)
win.run()
win.run()
torch.cuda.synchronize()
print("ok")
