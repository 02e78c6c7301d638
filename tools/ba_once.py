"""One NEXT-4 BA iteration over the C5 keyframe DB (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200.ba import gpu_ba  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402

dev = torch.device("cuda:0")
sc = synth.window_scene(0)
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
st.size_pairs(sc.views[0], views=sc.views[1:4])
st.prepare()
oc, od = [], []
for v in sc.views:
    st.project_bin(v)
    st.forward()
    oc.append(st.img["color"].clone())
    od.append(st.img["depth"].clone())
patches = synth.sample_patches(1, len(sc.views), sc.cam["width"], sc.cam["height"], 65536)
ba = gpu_ba(st, sc.views, oc, od, patches, rank=0, world=1)
ba.run()
torch.cuda.synchronize()
print("marker")
ba.run()
torch.cuda.synchronize()
print("ok")
